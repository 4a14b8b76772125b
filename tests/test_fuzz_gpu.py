"""Seeded fuzz of the sm_100a GEMM path: random ragged shapes x schedule space
(cta_group, tileN, tileK, stages, inner, WRAP/FUSED, B layout, out dtype,
batch), every case bit-exact against the exact integer product on the
reference's D-int inputs (SplitMix64 range(-8,8))."""
import random

import numpy as np
import pytest

from oracle.splitmix import gemm_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = 60


def _case(i):
    r = random.Random(1000 + i)
    cg = r.choice([1, 1, 2])
    tileN = r.choice([64, 128, 192, 256] if cg == 1 else [128, 192, 256])
    tileK = r.choice([32, 64, 128])
    st = r.randint(1, 6)
    inner = 1 if st == 1 else r.choice([1, 2])
    mode = r.choice([0, 1])
    layout = r.choice([0, 1])
    out = r.choice(["f32", "bf16", "f16"])
    batch = r.choice([1, 1, 1, 2, 3])
    M = r.randint(1, 700)
    N = r.randint(1, 640) // 8 * 8 + 8
    K = r.randint(1, 600) // 8 * 8 + 8
    return dict(cg=cg, tileN=tileN, tileK=tileK, st=st, inner=inner, mode=mode, layout=layout, out=out,
                batch=batch, M=M, N=N, K=K)


@pytest.mark.parametrize("i", range(CASES))
def test_fuzz_exact(alcop, i):
    _run_case(alcop, _case(i), i)


def _run_case(alcop, c, i):
    in_dt = torch.float16 if c["out"] == "f16" else torch.bfloat16
    out_dt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[c["out"]]
    s = alcop.make_schedule(tileN=c["tileN"], tileK=c["tileK"], n_stage=c["st"], n_stage_inner=c["inner"],
                            mode=c["mode"], cta_group=c["cg"])
    d = alcop.gemm_desc(c["M"], c["N"], c["K"], c["batch"], alcop.F16 if in_dt == torch.float16 else alcop.BF16,
                        {"f32": alcop.F32, "bf16": alcop.BF16, "f16": alcop.F16}[c["out"]],
                        alcop.B_KN if c["layout"] == 0 else alcop.B_NK)
    try:
        alcop.validate(d, s)
    except alcop.AlcopError:
        pytest.skip("schedule invalid for this case (checked by the rule tests)")
    a, b = gemm_inputs(c["M"], c["N"], c["K"], c["batch"], seed=i)
    # float64 BLAS product: exact for D-int inputs (|sum| <= 64 K << 2^53), far faster than an int64 matmul
    exact = np.rint(np.matmul(a.astype(np.float64), b.astype(np.float64))).astype(np.int64)
    A = torch.from_numpy(a).to(in_dt).cuda()
    Bt = torch.from_numpy(b).to(in_dt)
    if c["layout"] == 1:
        Bt = Bt.transpose(-1, -2).contiguous()
    C = alcop.matmul(A, Bt.cuda(), s, out_dtype=out_dt, b_layout=alcop.B_KN if c["layout"] == 0 else alcop.B_NK)
    torch.cuda.synchronize()
    ref = torch.from_numpy(exact.astype(np.float64)).to(torch.float32)
    if out_dt != torch.float32:
        ref = ref.to(out_dt)
    got = C.cpu()
    if not torch.equal(got, ref):
        bad = int((got.float() != ref.float()).sum())
        raise AssertionError("case %s: %d mismatches" % (c, bad))


def _pair_case(i):
    """CTA-pair schedules only, the 256 x 512 tile included (one 512-column
    TMEM accumulator: inner 1), larger ragged shapes."""
    r = random.Random(5000 + i)
    tileN = r.choice([128, 192, 256, 512, 512])
    tileK = r.choice([32, 64, 128])
    st = r.randint(1, 8)
    inner = 1 if (tileN == 512 or st == 1) else r.choice([1, 2])
    return dict(cg=2, tileN=tileN, tileK=tileK, st=st, inner=inner, mode=r.choice([0, 1]), layout=r.choice([0, 1]),
                out=r.choice(["f32", "bf16", "f16"]), batch=r.choice([1, 1, 2]), M=r.randint(1, 1300),
                N=r.randint(1, 1100) // 8 * 8 + 8, K=r.randint(1, 900) // 8 * 8 + 8)


@pytest.mark.parametrize("i", range(40))
def test_fuzz_pairs_exact(alcop, i):
    _run_case(alcop, _pair_case(i), 100 + i)
