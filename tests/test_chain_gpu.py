"""GPU parity of alcop_gemm_chain: several GEMMs in one persistent launch.

Independent problems (dep 0) must each equal the exact integer product; a
real data chain (A_p IS the buffer C_{p-1}, dep 1) must equal the chain
computed on the host with the same roundings — a row block read before its
producer stored it would show up as a mismatch.
"""
import numpy as np
import pytest

from oracle.splitmix import gemm_inputs

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bf16_round(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.float32).to(torch.bfloat16)


@pytest.mark.parametrize("tileN,tileK,st,cg", [(192, 64, 5, 1), (256, 64, 4, 1), (128, 128, 3, 1), (64, 32, 6, 1),
                                               (256, 64, 6, 2), (128, 64, 7, 2), (256, 128, 3, 2)])
def test_chain_independent_exact(alcop, tileN, tileK, st, cg):
    shapes = [(512, 384, 256), (384, 192, 640), (640, 576, 128), (256, 128, 64)]
    gemms, want = [], []
    for i, (M, N, K) in enumerate(shapes):
        a, b = gemm_inputs(M, N, K, seed=20 + i)
        want.append(torch.from_numpy((a.astype(np.int64) @ b.astype(np.int64)).astype(np.float64)).float())
        gemms.append((torch.from_numpy(a).to(torch.bfloat16).cuda(), torch.from_numpy(b).to(torch.bfloat16).cuda(),
                      torch.zeros((M, N), dtype=torch.float32, device="cuda")))
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=st, cta_group=cg)
    alcop.gemm_chain(gemms, s)
    torch.cuda.synchronize()
    for (A, B, C), w in zip(gemms, want):
        assert torch.equal(C.cpu(), w)


@pytest.mark.parametrize("M", [4096, 1000])
@pytest.mark.parametrize("layout", [0, 1], ids=["KN", "NK"])
@pytest.mark.parametrize("cg", [1, 2], ids=["cta", "pair"])
def test_chain_dependent_exact(alcop, M, layout, cg):
    """X @ W0 -> C0 (bf16) -> C0 @ W1 -> C1 -> C1 @ W2 -> C2: each A_p is the
    previous C buffer.  Integer data: every fp32 sum is exact; the bf16
    output rounding is reproduced on the host."""
    Ks = [128, 192, 256, 64]  # K0, N0 = K1, N1 = K2, N2
    rng = np.random.default_rng(7)
    x = rng.integers(-2, 3, size=(M, Ks[0])).astype(np.float64)
    ws = [rng.integers(-2, 3, size=(Ks[i], Ks[i + 1])).astype(np.float64) for i in range(3)]
    X = torch.from_numpy(x).to(torch.bfloat16).cuda()
    Cs = [torch.zeros((M, Ks[i + 1]), dtype=torch.bfloat16, device="cuda") for i in range(3)]
    Ws = []
    for w in ws:
        t = torch.from_numpy(w).to(torch.bfloat16)
        Ws.append((t if layout == 0 else t.t().contiguous()).cuda())
    gemms = [(X, Ws[0], Cs[0]), (Cs[0], Ws[1], Cs[1]), (Cs[1], Ws[2], Cs[2])]
    # (CTA pairs: 256-row blocks, half of the 128 tile columns per CTA; M = 1000: a ragged last pair tile)
    s = alcop.make_schedule(tileN=64 * cg, tileK=64, n_stage=4, cta_group=cg)
    for _ in range(3):  # repeated launches: stale counters or early reads would show
        for c in Cs:
            c.zero_()
        alcop.gemm_chain(gemms, s, dep=[0, 1, 1], b_layout=alcop.B_KN if layout == 0 else alcop.B_NK)
        torch.cuda.synchronize()
        ref = x
        for i, w in enumerate(ws):
            ref = _bf16_round(ref @ w).double().numpy()
            assert torch.equal(Cs[i].cpu(), _bf16_round(ref)), "chain step %d" % i


def test_chain_rejects_bad_dependency(alcop):
    a = torch.zeros((256, 64), dtype=torch.bfloat16, device="cuda")
    b = torch.zeros((64, 64), dtype=torch.bfloat16, device="cuda")
    c = torch.zeros((128, 64), dtype=torch.bfloat16, device="cuda")
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=2)
    with pytest.raises(alcop.AlcopError):
        alcop.gemm_chain([(a, b, a.new_zeros((256, 64))), (c[:, :64].contiguous(), b, c)], s, dep=[0, 1])


def test_chain_pair_rejects_split_atoms(alcop):
    """A chain on CTA pairs with B[K,N] stages whole 64-column atoms per CTA:
    tileN 192 (96 columns per CTA) is named, not run."""
    a = torch.zeros((256, 64), dtype=torch.bfloat16, device="cuda")
    b = torch.zeros((64, 192), dtype=torch.bfloat16, device="cuda")
    s = alcop.make_schedule(tileN=192, tileK=64, n_stage=4, cta_group=2)
    with pytest.raises(alcop.AlcopError, match="Unsupported"):
        alcop.gemm_chain([(a, b, a.new_zeros((256, 192)))], s)


@pytest.mark.parametrize("seed", range(24))
def test_chain_fuzz(alcop, seed):
    """Seeded chains: 2-4 GEMMs, random ragged M (shared when dependent) / N / K, a real data chain (A_p IS
    C_{p-1}) where dep[p] = 1, one CTA or a CTA pair per tile, both B layouts; bit-exact against the
    host chain with the same bf16 roundings."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(2, 5))
    cg = int(rng.integers(1, 3))
    layout = int(rng.integers(0, 2))
    tileN = int(rng.choice([128, 256])) if cg == 2 else int(rng.choice([64, 128, 192, 256]))
    tileK = int(rng.choice([32, 64, 128]))
    st = int(rng.integers(2, 6))
    M = int(rng.integers(1, 1300))
    dep = [0] + [int(rng.integers(0, 2)) for _ in range(n - 1)]
    dims = [int(rng.integers(1, 40)) * 8 for _ in range(n + 1)]  # K_0, N_0 = K_1 (when chained), ...
    gemms, refs = [], []
    prev_c, prev_ref = None, None
    for p in range(n):
        K, N = dims[p], dims[p + 1]
        if dep[p]:
            A, a = prev_c, prev_ref  # the previous C buffer is this A (K = N_{p-1})
        else:
            a = rng.integers(-2, 3, size=(M, K)).astype(np.float64)
            A = torch.from_numpy(a).to(torch.bfloat16).cuda()
        w = rng.integers(-2, 3, size=(K, N)).astype(np.float64)
        Wt = torch.from_numpy(w).to(torch.bfloat16)
        C = torch.zeros((M, N), dtype=torch.bfloat16, device="cuda")
        ref = _bf16_round(a @ w).double().numpy()
        gemms.append((A, (Wt if layout == 0 else Wt.t().contiguous()).cuda(), C))
        refs.append(ref)
        prev_c, prev_ref = C, ref
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=st, cta_group=cg)
    try:
        alcop.gemm_chain(gemms, s, dep=dep, b_layout=alcop.B_KN if layout == 0 else alcop.B_NK)
    except alcop.AlcopError as e:
        assert any(t in str(e) for t in ("SmemCapacity", "BadTile", "Unsupported", "BadStages")), (s, e)
        pytest.skip("schedule invalid for this chain: %s" % e)
    torch.cuda.synchronize()
    for p, ((_, _, C), ref) in enumerate(zip(gemms, refs)):
        assert torch.equal(C.cpu(), _bf16_round(ref)), "chain %s dep %s, GEMM %d, %s" % (dims, dep, p, s)
