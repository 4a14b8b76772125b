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
    assert bench.step_flops() == sum(2.0 * M * N * K for _, M, N, K in bench.BERT_GEMMS)
    # the fused-QKV step has the same FLOPs as the six-GEMM layer
    assert bench.step_flops() == sum(2.0 * M * N * K for _, M, N, K in bench.BERT_GEMMS_UNFUSED)


@pytest.mark.skipif(bench._ref_driver() is None, reason="oracle/_ref not built")
def test_reference_sample_runs():
    dt, flops, kind, cores = bench.cpu_reference_step(1)
    assert kind == "reference" and dt > 0 and cores >= 1
    assert flops == sum(2.0 * 1 * bench.REF_SAMPLE_COLS * K
                        for j in range(max(len(bench.BERT_GEMMS), os.cpu_count() or 1))
                        for K in [bench.BERT_GEMMS[j % len(bench.BERT_GEMMS)][3]])


@pytest.mark.skipif(bench._ref_driver() is None, reason="oracle/_ref not built")
def test_reference_arm_line():
    out = subprocess.run([sys.executable, "-c",
                          "import bench; bench.ref_sample_rows = lambda s: 1; import sys; "
                          "sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '3']; "
                          "bench.main()"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "cpu_baseline", "e2e"):
        assert key in line
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
