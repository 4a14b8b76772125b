"""The drop-in boundary: libalcop.so loads without a GPU, exports every
function include/alcop.h declares, and rejects bad schedules with the
reference's exit-code numbering (cli.hpp:23-25) and rule tags."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "alcop.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(alcop_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(alcop):
    lib = alcop.load_library()
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(alcop.EXPORTED_SYMBOLS)


def test_version_and_error_string(alcop):
    assert "sm_100a" in alcop.version()


@pytest.mark.parametrize("field,value,rule", [
    ("tileM", 64, "BadTile"), ("tileN", 96, "BadTile"), ("tileK", 16, "BadTile"),
    ("n_stage_smem_A", 0, "BadStages"), ("n_stage_inner", 3, "BadStages"), ("mode", 7, "BadSchedule"),
    ("raster", -1, "BadRaster"),
    ("cta_group", 4, "BadSchedule"),
    ("stream_k", 1, "BadSchedule"),  # stream-K needs cta_group 2 (make_schedule default: 1)
    ("stream_k", 2, "BadSchedule"),
])
def test_validate_rejects(alcop, field, value, rule):
    d = alcop.gemm_desc(1024, 1024, 1024)
    s = alcop.make_schedule()
    setattr(s, field, value)
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.validate(d, s)
    assert ei.value.code == alcop.ALCOP_ERR_CONFIG
    assert ei.value.rule == rule


def test_validate_capacity_and_lookahead(alcop):
    d = alcop.gemm_desc(1024, 1024, 1024)
    s = alcop.make_schedule(tileN=256, tileK=128, n_stage=4)
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.validate(d, s)
    assert ei.value.rule == "SmemCapacity"
    s = alcop.make_schedule(tileN=256, tileK=64, n_stage=4, n_stage_inner=2)
    alcop.validate(d, s)
    assert alcop.smem_bytes(d, s) <= 232448
    # TMA needs 16-byte row pitch
    with pytest.raises(alcop.AlcopError) as ei:
        alcop.validate(alcop.gemm_desc(128, 128, 100), s)
    assert ei.value.rule == "Alignment"


def test_null_arguments(alcop):
    lib = alcop.load_library()
    assert lib.alcop_gemm(None, None, None, None, None, None) == alcop.ALCOP_ERR_CONFIG
    assert lib.alcop_last_error().decode().startswith("NullArgument")


def test_host_entry_rejects_strided(alcop):
    lib = alcop.load_library()
    d = alcop.gemm_desc(128, 128, 128, ldc=256)
    s = alcop.make_schedule()
    dummy = ctypes.c_void_p(16)
    rc = lib.alcop_gemm_host(ctypes.byref(d), ctypes.byref(s), dummy, dummy, dummy, dummy, None)
    assert rc == alcop.ALCOP_ERR_CONFIG


@pytest.mark.parametrize("cg,sk,c", [(2, 0, 24), (2, 1, 64), (1, 1, 64)])
def test_conv_rejects_pair_and_stream_k(alcop, cg, sk, c):
    """the conv kernels run whole tiles (no stream-K), and
    CTA pairs only on the 64-channel im2col path; other schedules are
    rejected before any launch."""
    lib = alcop.load_library()
    d = alcop.conv_desc(2, 14, 14, c, 128, 3, 3, (2, 2), (1, 1))
    s = alcop.make_schedule(tileN=256, tileK=64, n_stage=4, cta_group=cg, stream_k=sk)
    dummy = ctypes.c_void_p(256)
    rc = lib.alcop_conv2d(ctypes.byref(d), ctypes.byref(s), dummy, dummy, dummy, None)
    assert rc == alcop.ALCOP_ERR_CONFIG
    assert lib.alcop_last_error().decode().startswith("BadSchedule")


def test_pre_op_model_pick_is_valid(alcop):
    """the model's pick for a pre-op GEMM comes from the space valid
    for the pre-op kernel (cta_group 1, its shared-memory budget)."""
    for shape in ((4096, 4096, 4096), (4096, 3072, 768), (4096, 768, 3072), (512, 512, 512)):
        d = alcop.gemm_desc(*shape, pre_op=1)
        s = alcop.choose_schedule(d)
        assert s.cta_group == 1
        alcop.validate(d, s)


def test_matmul_checks_operands(alcop):
    """shapes, dtypes and `out` are checked before the descriptor is
    built (no silent out-of-bounds reads from a mismatched B)."""
    torch = pytest.importorskip("torch")
    A = torch.zeros(3, 64, 32, dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="both be 2-D or both 3-D"):
        alcop.matmul(A, torch.zeros(32, 16, dtype=torch.bfloat16))
    with pytest.raises(ValueError, match="reduction sizes"):
        alcop.matmul(A, torch.zeros(3, 48, 16, dtype=torch.bfloat16))
    with pytest.raises(ValueError, match="batch sizes"):
        alcop.matmul(A, torch.zeros(2, 32, 16, dtype=torch.bfloat16))
    with pytest.raises(TypeError, match="dtypes differ"):
        alcop.matmul(A, torch.zeros(3, 32, 16, dtype=torch.float16))
    with pytest.raises(ValueError, match="out has shape"):
        alcop.matmul(A, torch.zeros(3, 32, 16, dtype=torch.bfloat16), out=torch.zeros(3, 64, 8))
    with pytest.raises(TypeError, match="out dtype"):
        alcop.matmul(A, torch.zeros(3, 32, 16, dtype=torch.bfloat16), out=torch.zeros(3, 64, 16),
                     out_dtype=torch.bfloat16)
    with pytest.raises(ValueError, match="reduction sizes"):
        alcop.matmul(A[0], torch.zeros(16, 48, dtype=torch.bfloat16), b_layout=alcop.B_NK)
