"""CPU checks of bench.py's host-side pieces: the config-1 script it times is the
reference's own BASELINE schedule, the reference CPU arm's sample runs through
the compiled reference interpreter, and the reference arm prints the contract
line."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_config1_script_is_the_baseline_schedule(alcop):
    d = alcop.gemm_desc(512, 512, 512, 1, alcop.F16, alcop.F16, alcop.B_KN)
    script = bench._ref_sample_script(128, 128, 512).replace("i0=1", "i0=4").replace("j0=1", "j0=4")
    s, warns = alcop.apply_script(d, script)
    assert not warns
    assert (s.tileM, s.tileN, s.tileK, s.n_stage_smem_A, s.n_stage_smem_B, s.n_stage_inner, s.mode) == \
        (128, 128, 32, 2, 2, 2, alcop.MODE_WRAP)


def test_step_flops():
    assert bench.step_flops() == sum(2.0 * n ** 3 for n in (4096, 8192, 12288, 16384))
    # the fused-QKV BERT step has the same FLOPs as the six-GEMM layer
    assert bench.bert_step_flops() == sum(2.0 * M * N * K for _, M, N, K in bench.BERT_GEMMS_UNFUSED)


@pytest.mark.skipif(bench._ref_driver() is None, reason="oracle/_ref not built")
def test_reference_sample_runs():
    dt, flops, kind, cores = bench.cpu_reference_step(1, sizes=(256, 512))
    assert kind == "reference" and dt > 0 and cores >= 1
    nproc = max(2, os.cpu_count() or 1)
    assert flops == sum(2.0 * 1 * bench.REF_SAMPLE_COLS * (256, 512)[j % 2] for j in range(nproc))


@pytest.mark.skipif(bench._ref_driver() is None, reason="oracle/_ref not built")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, "-c",
                          "import bench; bench.ref_sample_rows = lambda s: 1; bench.SQUARES = (256, 512); "
                          "import sys; "
                          "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']; "
                          "bench.main()"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e"):
        assert key in line
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"


def _run_dry(world, extra=()):
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(world), "--dry-run",
                          "--steps", "3", "--warmup", "3", "--no-cpu"] + list(extra),
                         cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])


@pytest.mark.parametrize("world", [1, 2])
def test_bench_rank_logic_dry_run(world):
    """bench.py --gpus N launches N ranks itself (torch.distributed.run, gloo in
    the dry run), shards every square's rows in 256-row granules (scaled) with
    no overlap and full cover, times with barrier + max over ranks and prints
    ONE contract line from rank 0."""
    line = _run_dry(world)
    assert line["n_gpus"] == world and line["dry_run"] and line["scaling"] == "strong"
    assert line["steps"] == 3 and line["warmup"] == 3 and line["value"] > 0
    assert line["parity"]["all_exact"]
    assert len(line["parity"]["checks"]) == 4 * world
    for i, n_full in enumerate(bench.SQUARES):
        n = n_full // bench.DRY_SCALE
        spans = sorted(tuple(r[str(n_full)]) for r in line["shards"])
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all((b - a) % (bench.SQUARE_GRANULE // bench.DRY_SCALE) == 0 for a, b in spans[:-1])


def test_bench_rejects_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
