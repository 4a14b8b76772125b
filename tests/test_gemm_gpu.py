"""GPU parity of the sm_100a pipelined GEMM/BMM kernels (through the C ABI).

D-int inputs (SplitMix64 range(-8,8), the reference generator) are exact in
fp16/bf16 and every fp32 partial sum is an integer < 2^24, so the kernel's
fp32 output must equal the exact integer product bit-for-bit, and bf16/f16
output must equal its round-to-nearest-even value bit-for-bit.  D-float
inputs are checked against a float64 reference with the tolerance stated in
SURVEY §8(d): |d| <= 2 ulp(out)*|ref| + 2^-20*sqrt(K)  (rel. Frobenius 1e-5
for fp32 out).
"""
import numpy as np
import pytest

from oracle.splitmix import gemm_inputs, uniform_tensor

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _exact(a, b, batched):
    # float64 BLAS product: exact for D-int inputs (|sum| <= 64 K << 2^53), far faster than an int64 matmul
    return np.rint(np.matmul(a.astype(np.float64), b.astype(np.float64))).astype(np.int64)


def _run(alcop, M, N, K, batch=1, in_dt=None, out_dt=None, b_layout=0, sched=None, seed=0):
    in_dt = in_dt or torch.bfloat16
    out_dt = out_dt or torch.float32
    a, b = gemm_inputs(M, N, K, batch, seed=seed)
    exact = _exact(a, b, batch > 1)
    A = torch.from_numpy(a).to(in_dt).cuda()
    Bt = torch.from_numpy(b).to(in_dt)
    if b_layout == alcop.B_NK:
        Bt = Bt.transpose(-1, -2).contiguous()
    B = Bt.cuda()
    C = alcop.matmul(A, B, sched, out_dtype=out_dt, b_layout=b_layout)
    torch.cuda.synchronize()
    return C.cpu(), exact


def _assert_exact(C, exact, out_dt):
    ref = torch.from_numpy(exact.astype(np.float64))
    if out_dt == torch.float32:
        ref = ref.to(torch.float32)
    else:
        ref = ref.to(torch.float32).to(out_dt)  # exact int -> fp32 exact -> RNE to out dtype
    if not torch.equal(C, ref):
        diff = (C.float() - ref.float()).abs()
        idx = torch.nonzero(diff)[:5]
        raise AssertionError("mismatch at %s: got %s want %s (n=%d)" %
                             (idx.tolist(), [C[tuple(i)].item() for i in idx],
                              [ref[tuple(i)].item() for i in idx], int((diff != 0).sum())))


@pytest.mark.parametrize("mode", [0, 1], ids=["wrap", "fused"])
def test_config1_fp16_512_exact(alcop, mode):
    """BASELINE config 1: fp16 512^3, tile 128x128x32, 2 smem + 2 inner stages."""
    s = alcop.make_schedule(tileN=128, tileK=32, n_stage=2, n_stage_inner=2, mode=mode)
    C, exact = _run(alcop, 512, 512, 512, in_dt=torch.float16, out_dt=torch.float32, sched=s)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("tileN", [64, 128, 192, 256])
@pytest.mark.parametrize("tileK", [32, 64, 128])
def test_tiles_exact(alcop, tileN, tileK):
    stage_bytes = (128 + tileN) * tileK * 2
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=min(3, 220000 // stage_bytes), n_stage_inner=2)
    C, exact = _run(alcop, 256, 3 * 192 if tileN == 192 else 512, 384, sched=s)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("sA,sB,inner", [(1, 1, 1), (2, 2, 1), (1, 3, 2), (4, 2, 2), (5, 5, 2), (6, 6, 2), (8, 7, 2)])
@pytest.mark.parametrize("mode", [0, 1], ids=["wrap", "fused"])
def test_stages_exact(alcop, sA, sB, inner, mode):
    s = alcop.make_schedule(tileN=128, tileK=64 if max(sA, sB) < 7 else 32, n_stage=sA, n_stage_B=sB, n_stage_inner=inner, mode=mode)
    C, exact = _run(alcop, 384, 384, 640, sched=s)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("out_dt", ["bf16", "f16"])
def test_half_output_rne(alcop, out_dt):
    odt = torch.bfloat16 if out_dt == "bf16" else torch.float16
    idt = torch.bfloat16 if out_dt == "bf16" else torch.float16
    s = alcop.make_schedule(tileN=256, tileK=64, n_stage=4)
    C, exact = _run(alcop, 512, 768, 768, in_dt=idt, out_dt=odt, sched=s)
    _assert_exact(C, exact, odt)


def test_b_layout_nk(alcop):
    for tk in (32, 64, 128):
        s = alcop.make_schedule(tileN=128, tileK=tk, n_stage=3)
        C, exact = _run(alcop, 256, 256, 512, b_layout=alcop.B_NK, sched=s)
        _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("mode", [0, 1], ids=["wrap", "fused"])
def test_batched_exact(alcop, mode):
    s = alcop.make_schedule(tileN=128, tileK=64, n_stage=3, mode=mode)
    C, exact = _run(alcop, 256, 128, 192, batch=5, sched=s)
    _assert_exact(C, exact, torch.float32)


def test_ragged_shapes(alcop):
    # M, N not multiples of the tile; K not a multiple of tileK (TMA zero fill)
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=3)
    C, exact = _run(alcop, 300, 200, 104, sched=s)
    _assert_exact(C, exact, torch.float32)
    s = alcop.make_schedule(tileN=128, tileK=32, n_stage=2)
    C, exact = _run(alcop, 130, 136, 40, batch=3, sched=s)
    _assert_exact(C, exact, torch.float32)


def test_single_tile_many_ctas(alcop):
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=2)
    C, exact = _run(alcop, 128, 64, 64, sched=s)
    _assert_exact(C, exact, torch.float32)


def test_float_inputs_tolerance(alcop):
    M, N, K = 1024, 768, 3072
    a = uniform_tensor(M * K, 11).reshape(M, K)
    b = uniform_tensor(K * N, 12).reshape(K, N)
    A = torch.from_numpy(a).to(torch.bfloat16)
    B = torch.from_numpy(b).to(torch.bfloat16)
    ref = A.double() @ B.double()
    s = alcop.make_schedule(tileN=256, tileK=64, n_stage=4)
    C32 = alcop.matmul(A.cuda(), B.cuda(), s, out_dtype=torch.float32).cpu().double()
    rel = (C32 - ref).norm() / ref.norm()
    assert rel < 1e-5, rel
    Cb = alcop.matmul(A.cuda(), B.cuda(), s, out_dtype=torch.bfloat16).cpu().double()
    ulp = 2.0 ** -7
    tol = 2 * ulp * ref.abs() + 2.0 ** -20 * np.sqrt(K)
    assert bool(((Cb - ref).abs() <= tol).all())


@pytest.mark.parametrize("mode", [0, 1], ids=["wrap", "fused"])
@pytest.mark.parametrize("sA,sB", [(2, 2), (3, 2), (1, 4)])
def test_device_trace_matches_enumerator(alcop, mode, sA, sB):
    """Bit-exact stage bookkeeping: every CTA's producer and MMA-thread event
    stream equals the host enumerator (which tests/test_bookkeeping.py pins to
    the reference pass + interpreter)."""
    s = alcop.make_schedule(tileN=64, tileK=64, n_stage=sA, n_stage_B=sB, n_stage_inner=2, mode=mode, num_ctas=3)
    M, N, K = 256, 256, 320  # 8 tiles over 3 CTAs, E = 5
    a, b = gemm_inputs(M, N, K)
    A = torch.from_numpy(a).to(torch.bfloat16).cuda()
    B = torch.from_numpy(b).to(torch.bfloat16).cuda()
    C, traces = alcop.matmul_traced(A, B, s, out_dtype=torch.float32)
    _assert_exact(C.cpu(), _exact(a, b, False), torch.float32)
    tiles = 8
    for cta, (prod, cons) in enumerate(traces):
        my = (tiles - cta + 2) // 3
        # per-buffer streams (with equal stage counts the kernel guards A and
        # B of a chunk with one barrier pair, which interleaves the two
        # buffers' prologue events; each buffer's own sequence is unchanged)
        for b in (0, 1):
            want_p = [e for e in alcop.enumerate_pipeline(my, 5, sA, sB, mode, 0) if e["buf"] == b]
            want_c = [e for e in alcop.enumerate_pipeline(my, 5, sA, sB, mode, 1) if e["buf"] == b]
            assert [e for e in prod if e["buf"] == b] == want_p, (cta, b)
            assert [e for e in cons if e["buf"] == b] == want_c, (cta, b)


@pytest.mark.parametrize("tileN,tileK,st,mode,layout", [(256, 64, 4, 1, 0), (128, 64, 4, 0, 0), (256, 128, 2, 1, 1),
                                                        (128, 32, 6, 1, 1), (256, 64, 1, 1, 0), (128, 64, 3, 0, 1),
                                                        (192, 64, 4, 1, 0), (192, 128, 2, 0, 0), (192, 32, 6, 1, 0),
                                                        (192, 64, 4, 1, 1), (192, 32, 5, 0, 1)])
def test_cta_pair_exact(alcop, tileN, tileK, st, mode, layout):
    """cta_group::2: a CTA pair computes 256 x tileN tiles (M=256 tcgen05.mma)."""
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=st, n_stage_inner=2 if st > 1 else 1, mode=mode,
                            cta_group=2)
    C, exact = _run(alcop, 768, 512, 640, b_layout=layout, sched=s)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("M,N,K,batch,tileK,st,mode,layout,out", [
    (768, 1024, 640, 1, 64, 4, 1, 0, "f32"), (768, 1024, 640, 1, 64, 4, 1, 1, "f32"),
    (512, 1536, 1024, 1, 64, 3, 0, 0, "bf16"), (300, 712, 200, 2, 64, 4, 1, 0, "f32"),
    (300, 712, 200, 2, 64, 4, 1, 1, "bf16"), (1024, 2048, 512, 1, 128, 2, 1, 0, "bf16"),
    (1024, 2048, 512, 1, 128, 2, 1, 1, "f32"), (256, 512, 64, 1, 32, 6, 1, 0, "f32"),
    (2048, 512, 4096, 1, 64, 4, 1, 0, "bf16"), (640, 1000, 96, 3, 32, 5, 0, 1, "f32")])
def test_cta_pair_wide_exact(alcop, M, N, K, batch, tileK, st, mode, layout, out):
    """CTA pair with tileN 512: a 256 x 512 tile as two N = 256 tcgen05.mma per
    k-step (each CTA stages columns 256g + 128 rank + [0,128) of B), one TMEM
    accumulator of 512 columns; ragged M / N / K, batched, both B layouts."""
    s = alcop.make_schedule(tileN=512, tileK=tileK, n_stage=st, n_stage_inner=1, mode=mode, cta_group=2)
    out_dt = torch.float32 if out == "f32" else torch.bfloat16
    C, exact = _run(alcop, M, N, K, batch=batch, b_layout=layout, sched=s, out_dt=out_dt, seed=M + N)
    _assert_exact(C, exact, out_dt)


def test_cta_pair_wide_rejections(alcop):
    d = alcop.gemm_desc(1024, 1024, 1024)
    for kw in (dict(cta_group=1, n_stage_inner=1), dict(cta_group=2, n_stage_inner=2),
               dict(cta_group=2, n_stage_inner=1, stream_k=1)):
        with pytest.raises(alcop.AlcopError) as ei:
            alcop.validate(d, alcop.make_schedule(tileN=512, tileK=64, n_stage=4, **kw))
        assert ei.value.rule in ("BadTile", "TmemCapacity", "SmemCapacity")


def test_cta_pair_ragged_batched(alcop):
    s = alcop.make_schedule(tileN=128, tileK=64, n_stage=4, cta_group=2)
    C, exact = _run(alcop, 300, 200, 136, batch=3, sched=s)
    _assert_exact(C, exact, torch.float32)
    C, exact = _run(alcop, 512, 768, 768, in_dt=torch.bfloat16, out_dt=torch.bfloat16, sched=s)
    _assert_exact(C, exact, torch.bfloat16)
    s = alcop.make_schedule(tileN=192, tileK=64, n_stage=5, cta_group=2)
    C, exact = _run(alcop, 1024, 768, 3072, in_dt=torch.bfloat16, out_dt=torch.bfloat16, sched=s)
    _assert_exact(C, exact, torch.bfloat16)
    C, exact = _run(alcop, 300, 200, 136, batch=3, sched=s)
    _assert_exact(C, exact, torch.float32)



@pytest.mark.parametrize("tileN,tileK,st,mode", [(128, 64, 4, 1), (256, 64, 4, 0), (64, 32, 3, 1), (192, 128, 2, 1),
                                                 (128, 64, 1, 1)])
def test_fused_preop_exact(alcop, tileN, tileK, st, mode):
    """C = (2A+1) @ B with f applied in shared memory between the TMA landing
    and the MMA (the reference's inline S2 case 2, mma_ewa)."""
    M, N, K = 384, 3 * tileN if tileN == 192 else 512, 320
    a, b = gemm_inputs(M, N, K, seed=4)
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=st, n_stage_inner=2 if st > 1 else 1, mode=mode)
    C = alcop.matmul(torch.from_numpy(a).to(torch.bfloat16).cuda(), torch.from_numpy(b).to(torch.bfloat16).cuda(),
                     s, out_dtype=torch.float32, pre_op=1)
    _assert_exact(C.cpu(), _exact(2 * a + 1, b, False), torch.float32)


@pytest.mark.parametrize("cg,raster,num_ctas", [(1, 3, 10), (1, 1, 7), (2, 3, 8), (2, 2, 6), (1, 0, 0), (2, 0, 0)])
def test_grouped_raster_exact(alcop, cg, raster, num_ctas):
    """Grouped tile rasterisation (raster rows per group, ragged last group)
    with several tiles per persistent CTA: every tile is visited exactly once."""
    s = alcop.make_schedule(tileN=128, tileK=64, n_stage=4, cta_group=cg, raster=raster, num_ctas=num_ctas)
    M = 7 * 128 * cg + 40  # 8 tile rows, last one ragged
    C, exact = _run(alcop, M, 5 * 128 - 24, 192, batch=2, sched=s)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("cg,tileN,tileK", [(1, 256, 128), (1, 192, 64), (2, 192, 64), (2, 256, 128), (2, 128, 128)])
def test_atom_views_batched(alcop, cg, tileN, tileK):
    """One 4-D TMA box per operand per chunk (atom-stacked views of A[.., K/64]
    and B[K, N/atom]) with a batch dimension: batch strides and the atom
    coordinates must land every swizzle atom where the per-atom loads would."""
    st = max(2, min(4, 200000 // ((128 + tileN // cg) * tileK * 2)))
    s = alcop.make_schedule(tileN=tileN, tileK=tileK, n_stage=st, cta_group=cg)
    C, exact = _run(alcop, 512, 768, 384, batch=3, sched=s, seed=11)
    _assert_exact(C, exact, torch.float32)


@pytest.mark.parametrize("M,N,K,batch,out", [(4096, 384, 256, 1, "f32"), (1000, 192, 128, 1, "bf16"),
                                             (256, 128, 64, 3, "f32"), (640, 256, 192, 1, "f32")])
def test_gemm_host_pipelined_exact(alcop, M, N, K, batch, out):
    """alcop_gemm_host (HOST buffers): A streamed in row blocks on a copy stream,
    each block multiplied as it lands, C blocks copied back on a second stream —
    the result must equal the exact integer product like the device-buffer call."""
    import ctypes
    a, b = gemm_inputs(M, N, K, batch, seed=5)
    exact = _exact(a, b, batch > 1)
    out_dt = torch.float32 if out == "f32" else torch.bfloat16
    A = torch.from_numpy(a).to(torch.bfloat16).pin_memory()
    B = torch.from_numpy(b).to(torch.bfloat16).pin_memory()
    C = torch.zeros(exact.shape, dtype=out_dt).pin_memory()
    d = alcop.gemm_desc(M, N, K, batch, alcop.BF16, alcop.F32 if out == "f32" else alcop.BF16, alcop.B_KN)
    s = alcop.choose_schedule(d)
    lib = alcop.load_library()
    ws = torch.empty(lib.alcop_gemm_workspace_bytes(ctypes.byref(d)), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    rc = lib.alcop_gemm_host(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                             ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                             ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    assert rc == 0, lib.alcop_last_error()
    _assert_exact(C, exact, out_dt)


def test_gemm_host_async_back_to_back_exact(alcop):
    """alcop_gemm_host_async called back to back with one workspace each (the
    bench's e2e step): call k+1's H2D overlaps call k's D2H; A blocks of >= 8 MB
    (a 20 MB A streams in 2 row blocks, the small ones in 1); every C exact."""
    import ctypes
    lib = alcop.load_library()
    st = torch.cuda.current_stream()
    calls = []
    for i, (M, N, K) in enumerate([(2048, 768, 768), (10240, 256, 1024), (512, 384, 128), (4096, 1536, 768)]):
        a, b = gemm_inputs(M, N, K, 1, seed=40 + i)
        A = torch.from_numpy(a).to(torch.bfloat16).pin_memory()
        B = torch.from_numpy(b).to(torch.bfloat16).pin_memory()
        C = torch.zeros((M, N), dtype=torch.float32).pin_memory()
        d = alcop.gemm_desc(M, N, K, 1, alcop.BF16, alcop.F32, alcop.B_KN)
        ws = torch.empty(lib.alcop_gemm_workspace_bytes(ctypes.byref(d)), dtype=torch.uint8, device="cuda")
        calls.append((d, alcop.choose_schedule(d), A, B, C, ws, _exact(a, b, False)))
    for rep in range(2):
        for d, s, A, B, C, ws, _ in calls:
            rc = lib.alcop_gemm_host_async(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(A.data_ptr()),
                                           ctypes.c_void_p(B.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                                           ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(st.cuda_stream))
            assert rc == 0, lib.alcop_last_error()
        torch.cuda.synchronize()
        for d, s, A, B, C, ws, exact in calls:
            _assert_exact(C, exact, torch.float32)
            C.zero_()


def test_gemm_host_async_chain_shared_workspace_exact(alcop):
    """alcop_gemm_host_async where call k's host C is call k+1's host A, all
    calls sharing ONE workspace: call k+1's H2D must wait for call
    k's kernels (workspace) and for its D2H (the host data).  B_k are
    permutation matrices, so every C is exact in bf16 and the final C is A_0
    with its columns permuted three times."""
    import ctypes
    lib = alcop.load_library()
    st = torch.cuda.current_stream()
    M, N = 24576, 768
    a, _ = gemm_inputs(M, N, N, 1, seed=71)
    rng = np.random.default_rng(3)
    perms = [rng.permutation(N) for _ in range(3)]
    hosts = [torch.from_numpy(a).to(torch.bfloat16).pin_memory()]
    Bs = []
    for p in perms:
        b = np.zeros((N, N), dtype=np.float32)
        b[p, np.arange(N)] = 1.0  # C[:, j] = A[:, p[j]]
        Bs.append(torch.from_numpy(b).to(torch.bfloat16).pin_memory())
        hosts.append(torch.full((M, N), -1.0, dtype=torch.bfloat16).pin_memory())
    d = alcop.gemm_desc(M, N, N, 1, alcop.BF16, alcop.BF16, alcop.B_KN)
    s = alcop.choose_schedule(d)
    ws = torch.empty(lib.alcop_gemm_workspace_bytes(ctypes.byref(d)), dtype=torch.uint8, device="cuda")
    for k in range(3):
        rc = lib.alcop_gemm_host_async(ctypes.byref(d), ctypes.byref(s), ctypes.c_void_p(hosts[k].data_ptr()),
                                       ctypes.c_void_p(Bs[k].data_ptr()), ctypes.c_void_p(hosts[k + 1].data_ptr()),
                                       ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(st.cuda_stream))
        assert rc == 0, lib.alcop_last_error()
    torch.cuda.synchronize()
    want = a
    for p in perms:
        want = want[:, p]
    assert torch.equal(hosts[3], torch.from_numpy(np.ascontiguousarray(want)).to(torch.bfloat16))


@pytest.mark.parametrize("N,K,tileN,out", [(512, 64, 256, "bf16"), (512, 64, 128, "f32"), (384, 128, 192, "bf16"),
                                           (320, 64, 64, "f32")])
def test_short_k_eight_epilogue_warps_exact(alcop, N, K, tileN, out):
    """Tiles whose main loop is <= 2 chunks drain with 8 epilogue warps (two per
    TMEM lane quarter, alternate column chunks; gemm_epi_warps): batched, ragged N."""
    out_dt = torch.float32 if out == "f32" else torch.bfloat16
    s = alcop.make_schedule(tileN=tileN, tileK=64, n_stage=4)
    C, exact = _run(alcop, 512, N, K, batch=5, out_dt=out_dt, sched=s, seed=17)
    _assert_exact(C, exact, out_dt)
