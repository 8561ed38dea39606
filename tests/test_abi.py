"""The C-ABI library loads, exports every symbol include/sage.h declares, and rejects bad
arguments before launching anything (runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_02170_b200 import build, sage
    build.build()
    return sage.lib()


def test_exports_match_header(L):
    from paper_2603_02170_b200 import sage
    hdr = open(os.path.join(ROOT, "include", "sage.h")).read()
    declared = set(re.findall(r"SAGE_API\s+[\w\s\*]+?\b(sage_\w+)\s*\(", hdr))
    assert declared == set(sage.SYMBOLS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.sage_version() == 1
    assert L.sage_status_string(4) == b"SAGE_ERR_WORKSPACE"


def test_sizes_and_invalid_params(L):
    from paper_2603_02170_b200.sage import make_params
    p = make_params(2, 3, 256, 64, causal=True)
    nctx = L.sage_ctx_bytes(ctypes.byref(p))
    # q_i8 + k_i8 + 2 scale arrays + mu_K, 256-byte aligned
    assert nctx >= 2 * 2 * 3 * 256 * 64 + 2 * 2 * 3 * 2 * 4 + 2 * 3 * 64 * 4
    pq = make_params(2, 3, 256, 64, q_smooth=True)
    assert L.sage_ctx_bytes(ctypes.byref(pq)) > nctx  # + mu_Q and the bias
    assert L.sage_workspace_bytes(ctypes.byref(p), 1) >= 2 * 3 * 256 * 64 * 4  # fp32 dQ accumulator
    for bad in (make_params(1, 1, 0, 64), make_params(1, 1, 32769, 64), make_params(1, 1, 128, 96),
                make_params(0, 1, 128, 64), make_params(1, 1, 128, 64, softmax_scale=-1.0)):
        assert L.sage_ctx_bytes(ctypes.byref(bad)) == 0
        assert L.sage_workspace_bytes(ctypes.byref(bad), 0) == 0
    # a ragged N (reading A33) is valid: the library's buffers pad each head to 128 ceil(N / 128) rows
    pr, pp = make_params(2, 3, 200, 64, q_smooth=True), make_params(2, 3, 256, 64, q_smooth=True)
    assert L.sage_ctx_bytes(ctypes.byref(pr)) == L.sage_ctx_bytes(ctypes.byref(pp))
    assert L.sage_workspace_bytes(ctypes.byref(pr), 1) == L.sage_workspace_bytes(ctypes.byref(pp), 1)
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 1, 1, 128))) == L.sage_ctx_bytes(ctypes.byref(make_params(1, 1, 128, 128)))
    bad = make_params(1, 1, 128, 64)
    bad.flags = 1 << 12
    assert L.sage_ctx_bytes(ctypes.byref(bad)) == 0


def _ctx(buf, nbytes, tag=0):
    from paper_2603_02170_b200.sage import SageCtxDesc
    return ctypes.byref(SageCtxDesc(buf, nbytes, tag))


def test_params_tag(L):
    """sage_params_tag: a non-zero hash that separates every field (the ctx check of sage_bwd)."""
    from paper_2603_02170_b200.sage import make_params
    base = make_params(2, 3, 256, 64, causal=True)
    t0 = L.sage_params_tag(ctypes.byref(base))
    assert t0 != 0 and t0 == L.sage_params_tag(ctypes.byref(make_params(2, 3, 256, 64, causal=True)))
    others = [make_params(1, 3, 256, 64, causal=True), make_params(2, 2, 256, 64, causal=True),
              make_params(2, 3, 384, 64, causal=True), make_params(2, 3, 256, 128, causal=True),
              make_params(2, 3, 256, 64), make_params(2, 3, 256, 64, causal=True, q_smooth=True),
              make_params(2, 3, 256, 64, causal=True, softmax_scale=0.2),
              make_params(2, 3, 256, 64, causal=True, p_u8=True), make_params(2, 3, 256, 64, causal=True, fp32_out=True),
              make_params(2, 3, 256, 64, causal=True, strides=(256 * 3 * 64, 64, 3 * 64))]
    tags = {L.sage_params_tag(ctypes.byref(o)) for o in others}
    assert t0 not in tags and len(tags) == len(others)
    assert L.sage_params_tag(ctypes.byref(make_params(1, 1, 128, 96))) == 0


def test_stride_validation(L):
    """sage_params strides (S:8(b) layouts): all zero = contiguous; otherwise multiples of 8 elements with the
    token stride >= d; the ctx / workspace sizes do not depend on the I/O layout (internal buffers are
    contiguous)."""
    from paper_2603_02170_b200.sage import make_params
    B, H, N, d = 2, 3, 256, 64
    n0 = L.sage_ctx_bytes(ctypes.byref(make_params(B, H, N, d)))
    bshd = (N * H * d, d, H * d)  # a [B, N, H, d] tensor viewed as [B, H, N, d]
    assert L.sage_ctx_bytes(ctypes.byref(make_params(B, H, N, d, strides=bshd))) == n0
    for bad in ((N * H * d, d, H * d + 4), (N * H * d, d, 32), (N * H * d, 0, H * d), (-8, d, H * d)):
        assert L.sage_ctx_bytes(ctypes.byref(make_params(B, H, N, d, strides=bad))) == 0, bad


def test_error_paths_do_not_launch(L):
    """Validation happens before any device access: fake (never dereferenced) pointers."""
    from paper_2603_02170_b200.sage import make_params
    p = make_params(1, 2, 256, 64)
    nctx = L.sage_ctx_bytes(ctypes.byref(p))
    nws = L.sage_workspace_bytes(ctypes.byref(p), 0)
    tag = L.sage_params_tag(ctypes.byref(p))
    A = ctypes.c_void_p(0x10000)
    mis = ctypes.c_void_p(0x10008)
    z = ctypes.c_void_p(0)
    S = ctypes.c_size_t
    bad = make_params(1, 2, 256, 96)
    C = _ctx(0x10000, nctx)
    assert L.sage_fwd(ctypes.byref(bad), A, A, A, A, A, C, A, S(nws), z) == 1
    assert L.sage_fwd(ctypes.byref(p), z, A, A, A, A, C, A, S(nws), z) == 1
    assert L.sage_fwd(ctypes.byref(p), A, A, A, A, A, None, A, S(nws), z) == 1
    assert L.sage_fwd(ctypes.byref(p), mis, A, A, A, A, C, A, S(nws), z) == 3
    assert L.sage_fwd(ctypes.byref(p), A, A, A, A, A, _ctx(0x10000, nctx - 1), A, S(nws), z) == 4
    assert L.sage_fwd(ctypes.byref(p), A, A, A, A, A, C, A, S(nws - 1), z) == 4
    nwb = L.sage_workspace_bytes(ctypes.byref(p), 1)
    Ct = _ctx(0x10000, nctx, tag)
    assert L.sage_bwd(ctypes.byref(p), A, A, A, A, Ct, A, A, A, A, S(nwb - 1), z) == 4
    assert L.sage_bwd(ctypes.byref(p), A, A, A, A, Ct, A, A, mis, A, S(nwb), z) == 3
    # a context the forward never filled (tag 0), or filled under other params, is refused
    assert L.sage_bwd(ctypes.byref(p), A, A, A, A, C, A, A, A, A, S(nwb), z) == 1
    other = L.sage_params_tag(ctypes.byref(make_params(1, 2, 256, 64, causal=True)))
    assert L.sage_bwd(ctypes.byref(p), A, A, A, A, _ctx(0x10000, nctx, other), A, A, A, A, S(nwb), z) == 1
    assert L.sage_debug_umma(8, 64, 128, A, A, A, z) == 1
    assert L.sage_debug_umma(1, 128, 96, A, A, A, z) == 1
    # one backward variant at a time: SAGE_DETERMINISTIC with SAGE_P_COLSCALE is rejected
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 2, 256, 64, deterministic=True, p_colscale=True))) == 0
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 2, 256, 64, deterministic=True, fine_bwd=True))) == 0
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 2, 256, 64, p_colscale=True))) == nctx
    # SAGE_FP32_OUT is valid alone, not with QK-norm
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 2, 256, 64, fp32_out=True))) == nctx
    assert L.sage_ctx_bytes(ctypes.byref(make_params(1, 2, 256, 64, fp32_out=True, qk_norm=True))) == 0
    # QK-norm params need the _qknorm entry points, which need gamma and eps > 0
    pn = make_params(1, 2, 256, 64, qk_norm=True)
    ncn = L.sage_ctx_bytes(ctypes.byref(pn))
    assert ncn > nctx  # + rstd of the X_q, X_k rows
    nwn = L.sage_workspace_bytes(ctypes.byref(pn), 0)
    Cn = _ctx(0x10000, ncn)
    assert L.sage_fwd(ctypes.byref(pn), A, A, A, A, A, Cn, A, S(nwn), z) == 1
    assert L.sage_bwd(ctypes.byref(pn), A, A, A, A, _ctx(0x10000, ncn, L.sage_params_tag(ctypes.byref(pn))),
                      A, A, A, A, S(1 << 30), z) == 1
    F = ctypes.c_float
    assert L.sage_fwd_qknorm(ctypes.byref(p), A, A, A, A, A, F(1e-6), A, A, C, A, S(nws), z) == 1
    assert L.sage_fwd_qknorm(ctypes.byref(pn), A, A, A, z, A, F(1e-6), A, A, Cn, A, S(nwn), z) == 1
    assert L.sage_fwd_qknorm(ctypes.byref(pn), A, A, A, A, A, F(0.0), A, A, Cn, A, S(nwn), z) == 1
    assert L.sage_fwd_qknorm(ctypes.byref(pn), A, A, A, mis, A, F(1e-6), A, A, Cn, A, S(nwn), z) == 3
    assert L.sage_fwd_qknorm(ctypes.byref(pn), A, A, A, A, A, F(1e-6), A, A, _ctx(0x10000, ncn - 1), A, S(nwn),
                             z) == 4
    assert L.sage_bwd_qknorm(ctypes.byref(pn), A, A, A, A, A, A, A, A, Cn, A, A, A, A, A, A, S(1 << 30), z) == 1
    assert L.sage_bwd_qknorm(ctypes.byref(pn), A, A, A, A, A, A, A, A, _ctx(0x10000, ncn, L.sage_params_tag(
        ctypes.byref(pn))), A, A, A, z, A, A, S(1 << 30), z) == 1
    # the tile dumps exist only in the test build (libsage_trace.so)
    assert L.sage_debug_dump(A, A, A, A, A, 1) == 2
    assert L.sage_debug_fwd_dump(A, A, A, A, 1) == 2


def test_trace_build_exports_the_same_abi():
    """libsage_trace.so (timelines, tile dumps) exports the same C ABI and validates dump args."""
    from paper_2603_02170_b200 import build, sage
    if not os.path.exists(build.TRACE_LIB):
        build.build(trace=True)
    T = ctypes.CDLL(build.TRACE_LIB)
    for name in sage.SYMBOLS:
        assert hasattr(T, name), name
    A, z = ctypes.c_void_p(0x10000), ctypes.c_void_p(0)
    T.sage_debug_dump.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_int]
    assert T.sage_debug_dump(A, A, z, A, A, 1) == 1
    assert T.sage_debug_dump(A, A, A, A, A, -1) == 1


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_no_fallback(L):
    """Valid arguments on a machine without an sm_100 device: an error status, never a CPU result."""
    from paper_2603_02170_b200.sage import make_params
    p = make_params(1, 2, 256, 64)
    A = ctypes.c_void_p(0x10000)
    S = ctypes.c_size_t
    st = L.sage_fwd(ctypes.byref(p), A, A, A, A, A, _ctx(0x10000, 1 << 30), A, S(1 << 30), ctypes.c_void_p(0))
    assert st in (5, 6)  # SAGE_ERR_CUDA / SAGE_ERR_ARCH


def test_product_does_not_import_oracle():
    """The product package never references oracle/ (the oracle is test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2603_02170_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src and "liboracle" not in src, f
