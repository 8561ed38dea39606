"""Thin Python binding of libsage.so (include/sage.h): argument marshalling only.

Every step of the SageBwd path runs in the CUDA kernels behind the C ABI; PyTorch
is used for device memory and streams.  There is no CPU or PyTorch fallback: if the
library cannot be loaded, every entry point raises.
"""
import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SAGE_LIB selects the profiling build (libsage_trace.so) for scripts/trace_bwd.py only.
LIB_PATH = os.environ.get("SAGE_LIB") or os.path.join(_HERE, "libsage.so")

SAGE_CAUSAL, SAGE_K_SMOOTH, SAGE_Q_SMOOTH, SAGE_P_U8, SAGE_QK_NORM, SAGE_DETERMINISTIC, SAGE_P_COLSCALE = \
    1, 2, 4, 8, 16, 32, 64
SAGE_FINE_BWD, SAGE_FP16, SAGE_FP32_OUT, SAGE_PV_FP8 = 128, 256, 512, 1024
_STATUS = {0: "SAGE_OK", 1: "SAGE_ERR_INVALID_VALUE", 2: "SAGE_ERR_UNSUPPORTED", 3: "SAGE_ERR_MISALIGNED",
           4: "SAGE_ERR_WORKSPACE", 5: "SAGE_ERR_CUDA", 6: "SAGE_ERR_ARCH"}

# exported symbols of include/sage.h
SYMBOLS = ("sage_ctx_bytes", "sage_workspace_bytes", "sage_params_tag", "sage_fwd", "sage_bwd", "sage_fwd_qknorm",
           "sage_bwd_qknorm", "sage_ctx_get_view", "sage_debug_fwd_dump", "sage_debug_dump_acc",
           "sage_ws_get_view", "sage_debug_umma", "sage_debug_trace", "sage_debug_dump", "sage_profile_enable", "sage_profile_read",
           "sage_status_string", "sage_last_cuda_error", "sage_version")


class SageParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads", ctypes.c_int32), ("seqlen", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("flags", ctypes.c_uint32), ("softmax_scale", ctypes.c_float),
                ("stride_b", ctypes.c_int64), ("stride_h", ctypes.c_int64), ("stride_n", ctypes.c_int64)]


class SageCtxDesc(ctypes.Structure):
    """include/sage.h sage_ctx: the caller-owned device buffer and the params tag sage_fwd writes."""
    _fields_ = [("buf", ctypes.c_void_p), ("bytes", ctypes.c_size_t), ("params_tag", ctypes.c_uint64)]


class SageCtxView(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("q_i8", "k_i8", "q_scale", "k_scale", "mu_k", "mu_q", "bias",
                                               "rstd_q", "rstd_k")]


class SageWsView(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("v_i8", "v_scale", "do_i8", "do_scale", "delta", "dq_acc")]


class SageError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libsage.so (raises if it is missing: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SageError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, S = ctypes.c_void_p, ctypes.c_size_t
        pp = ctypes.POINTER(SageParams)
        L.sage_ctx_bytes.argtypes = [pp]
        L.sage_ctx_bytes.restype = S
        L.sage_workspace_bytes.argtypes = [pp, ctypes.c_int]
        L.sage_workspace_bytes.restype = S
        pc = ctypes.POINTER(SageCtxDesc)
        L.sage_params_tag.argtypes = [pp]
        L.sage_params_tag.restype = ctypes.c_uint64
        L.sage_fwd.argtypes = [pp, P, P, P, P, P, pc, P, S, P]
        L.sage_bwd.argtypes = [pp, P, P, P, P, pc, P, P, P, P, S, P]
        L.sage_fwd_qknorm.argtypes = [pp, P, P, P, P, P, ctypes.c_float, P, P, pc, P, S, P]
        L.sage_bwd_qknorm.argtypes = [pp, P, P, P, P, P, P, P, P, pc, P, P, P, P, P, P, S, P]
        L.sage_debug_fwd_dump.argtypes = [P, P, P, P, ctypes.c_int]
        L.sage_debug_dump_acc.argtypes = [P, P, P, P, P]
        L.sage_ctx_get_view.argtypes = [pp, P, ctypes.POINTER(SageCtxView)]
        L.sage_ws_get_view.argtypes = [pp, ctypes.c_int, P, ctypes.POINTER(SageWsView)]
        L.sage_debug_umma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P]
        L.sage_debug_trace.argtypes = [P, S]
        L.sage_debug_dump.argtypes = [P, P, P, P, P, ctypes.c_int]
        L.sage_profile_enable.argtypes = [ctypes.c_int]
        L.sage_profile_read.argtypes = [ctypes.POINTER(ctypes.c_double)] * 2 + [ctypes.POINTER(ctypes.c_int64)] * 3
        L.sage_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


def use_library(path):
    """Switch this binding to another build of the same C ABI (tests: libsage_trace.so for
    sage_debug_dump); returns the previous path.  Workspaces are build-independent."""
    global _lib, LIB_PATH
    old = LIB_PATH
    LIB_PATH, _lib = path, None
    lib()
    return old


def _check(status, what):
    if status != 0:
        extra = f" (cudaError {lib().sage_last_cuda_error()})" if status == 5 else ""
        raise SageError(f"{what}: {_STATUS.get(status, status)}{extra}")


def make_params(batch, heads, seqlen, head_dim, causal=False, k_smooth=True, q_smooth=False, softmax_scale=None,
                p_u8=False, qk_norm=False, deterministic=False, p_colscale=False, fine_bwd=False, fp16=False,
                fp32_out=False, pv_fp8=False, strides=None):
    flags = (SAGE_CAUSAL if causal else 0) | (SAGE_K_SMOOTH if k_smooth else 0) | (SAGE_Q_SMOOTH if q_smooth else 0) | \
        (SAGE_P_U8 if p_u8 else 0) | (SAGE_QK_NORM if qk_norm else 0) | (SAGE_DETERMINISTIC if deterministic else 0) | \
        (SAGE_P_COLSCALE if p_colscale else 0) | (SAGE_FINE_BWD if fine_bwd else 0) | (SAGE_FP16 if fp16 else 0) | \
        (SAGE_FP32_OUT if fp32_out else 0) | (SAGE_PV_FP8 if pv_fp8 else 0)
    sb, sh, sn = (0, 0, 0) if strides is None else strides
    return SageParams(batch, heads, seqlen, head_dim, flags, 0.0 if softmax_scale is None else softmax_scale,
                      sb, sh, sn)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream, device=None):
    """The caller's stream, or the current stream of the tensors' device (not of the current device)."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_io(*ts):
    """CUDA [B, H, N, d] tensors of one I/O dtype (bf16, or fp16 with SAGE_FP16), shape and device."""
    ref = ts[0]
    for t in ts:
        if not (t.is_cuda and t.dtype in (torch.bfloat16, torch.float16) and t.dim() == 4):
            raise SageError("tensors must be CUDA bf16 or fp16 [B, H, N, d]")
        if t.shape != ref.shape or t.device != ref.device or t.dtype != ref.dtype:
            raise SageError("shape/device/dtype mismatch")


def _layout_ok(t):
    """The library's strided I/O layout: d contiguous, the other strides multiples of 8 elements, the token
    stride >= d, and a 16-byte aligned base."""
    sb, sh, sn, sd = t.stride()
    return sd == 1 and sn >= t.shape[3] and sb % 8 == 0 and sh % 8 == 0 and sn % 8 == 0 and t.data_ptr() % 16 == 0


def _io_layout(*ts):
    """(strides for sage_params or None, the tensors): ts share one layout the library can address directly
    (no copy), else all are made contiguous."""
    st = ts[0].stride()
    if all(t.stride() == st for t in ts) and all(_layout_ok(t) for t in ts):
        B, H, N, d = ts[0].shape
        if st == (H * N * d, N * d, d, 1):
            return None, ts
        return (st[0], st[1], st[2]), ts
    return None, tuple(t.contiguous() for t in ts)


def _to_layout(t, ref_stride):
    """t in the given [B, H, N, d] element strides (a copy only if it differs)."""
    if t.stride() == tuple(ref_stride):
        return t
    out = torch.empty_strided(t.shape, ref_stride, dtype=t.dtype, device=t.device)
    out.copy_(t)
    return out


def _check_out(t, shape, dtype, device, what, stride=None):
    """A caller-provided output: of the expected shape, dtype, device and strides (contiguous by default)."""
    ok_stride = t.is_contiguous() if stride is None else tuple(t.stride()) == tuple(stride)
    if not (t.is_cuda and ok_stride and tuple(t.shape) == tuple(shape) and t.dtype == dtype and t.device == device):
        raise SageError(f"{what}: expected a {dtype} {tuple(shape)} tensor (strides {stride or 'contiguous'}) on "
                        f"{device}, got {t.dtype} {tuple(t.shape)} strides {tuple(t.stride())} on {t.device}")


class SageCtx:
    """Forward->backward state (Alg. 2 inputs): the caller-owned ctx buffer, the params it was
    produced under and the params tag sage_fwd wrote (sage_bwd rejects a ctx from other params)."""

    def __init__(self, params, ctx, shape, io_stride=None):
        self.params, self.buf, self.shape = params, ctx, shape
        self.desc = SageCtxDesc(ctx.data_ptr(), ctx.numel(), 0)
        B, H, N, d = shape
        self.io_stride = tuple(io_stride) if io_stride is not None else (H * N * d, N * d, d, 1)

    @property
    def out_dtype(self):
        if self.params.flags & SAGE_FP32_OUT:
            return torch.float32
        return torch.float16 if self.params.flags & SAGE_FP16 else torch.bfloat16

    def view(self):
        """Device tensors of the context (Q^, K^, scales, mu_K, mu_Q, bias) -- no copies.  The per-row
        buffers have Np = 128 ceil(N / 128) rows per head (N ragged: rows N.. are padding, reading A33)."""
        v = SageCtxView()
        _check(lib().sage_ctx_get_view(ctypes.byref(self.params), _ptr(self.buf), ctypes.byref(v)), "ctx_view")
        B, H, N, d = self.shape
        T = -(-N // 128)
        N = T * 128
        base = self.buf.data_ptr()

        def sl(addr, n, dtype, shape):
            if not addr:
                return None
            off = addr - base
            nbytes = n * torch.empty((), dtype=dtype).element_size()
            return self.buf[off:off + nbytes].view(dtype).view(shape)
        out = dict(q_i8=sl(v.q_i8, B * H * N * d, torch.int8, (B, H, N, d)),
                   k_i8=sl(v.k_i8, B * H * N * d, torch.int8, (B, H, N, d)),
                   q_scale=sl(v.q_scale, B * H * T, torch.float32, (B, H, T)),
                   k_scale=sl(v.k_scale, B * H * T, torch.float32, (B, H, T)),
                   mu_k=sl(v.mu_k, B * H * d, torch.float32, (B, H, d)),
                   mu_q=sl(v.mu_q, B * H * T * d, torch.float32, (B, H, T, d)),
                   bias=sl(v.bias, B * H * T * N, torch.float32, (B, H, T, N)),
                   rstd_q=sl(v.rstd_q, B * H * N, torch.float32, (B, H, N)),
                   rstd_k=sl(v.rstd_k, B * H * N, torch.float32, (B, H, N)))
        return out


class Workspace:
    """Reusable scratch buffers (sage_workspace_bytes), grown on demand, one per (device, stream,
    direction): calls on different streams never share scratch, and a buffer replaced when it grows
    was only used on its own stream (the caching allocator hands it out again in stream order)."""

    def __init__(self):
        self.bufs = {}

    def get(self, params, backward, device, stream=None):
        n = lib().sage_workspace_bytes(ctypes.byref(params), int(backward))
        if n == 0:
            raise SageError("invalid sage_params")
        device = torch.device(device)
        if device.index is None:
            device = torch.device(device.type, torch.cuda.current_device())
        s = torch.cuda.current_stream(device) if stream is None else stream
        key = (str(device), s.cuda_stream, bool(backward))
        b = self.bufs.get(key)
        if b is None or b.numel() < n:
            with torch.cuda.stream(s):
                b = torch.empty(n, dtype=torch.uint8, device=device)
            self.bufs[key] = b
        return b


_ws = Workspace()


def ws_view(params, backward, ws):
    v = SageWsView()
    _check(lib().sage_ws_get_view(ctypes.byref(params), int(backward), _ptr(ws), ctypes.byref(v)), "ws_view")
    return v


def _out_dtype(io_dtype, fp32_out):
    return torch.float32 if fp32_out else io_dtype


def forward(q, k, v, causal=False, k_smooth=True, q_smooth=False, softmax_scale=None, out=None, lse=None,
            ctx=None, workspace=None, stream=None, p_u8=False, deterministic=False, p_colscale=False,
            fine_bwd=False, fp32_out=False, pv_fp8=False):
    """sage_fwd (Alg. 1): returns (o, lse, SageCtx).  q, k, v: CUDA bf16 (or fp16) [B, H, N, d].
    p_u8: the unsigned-P^ variant (SAGE_P_U8); deterministic: a bitwise reproducible backward
    (SAGE_DETERMINISTIC); p_colscale: per-key psi(P) in the backward (SAGE_P_COLSCALE); fine_bwd: per-key
    psi(P) and per-key / per-query psi(dS) (SAGE_FINE_BWD); fp32_out: O (and later dQ, dK, dV) in fp32
    (SAGE_FP32_OUT); pv_fp8: the forward's P^V^ in FP8 E4M3 (SAGE_PV_FP8).  The backward inherits them
    through the ctx."""
    _check_io(q, k, v)
    strides, (q, k, v) = _io_layout(q, k, v)
    B, H, N, d = q.shape
    dev = q.device
    p = make_params(B, H, N, d, causal, k_smooth, q_smooth, softmax_scale, p_u8, deterministic=deterministic,
                    p_colscale=p_colscale, fine_bwd=fine_bwd, fp16=q.dtype == torch.float16, fp32_out=fp32_out,
                    pv_fp8=pv_fp8, strides=strides)
    if q.numel() == 0 and d in (64, 128):
        # empty batch, heads or sequence: nothing to compute (the C ABI rejects empty shapes), empty results
        o = torch.empty_strided(q.shape, q.stride(), dtype=_out_dtype(q.dtype, fp32_out), device=dev)
        return o, torch.empty((B, H, N), dtype=torch.float32, device=dev), \
            SageCtx(p, torch.empty(0, dtype=torch.uint8, device=dev), (B, H, N, d), q.stride())
    nctx = lib().sage_ctx_bytes(ctypes.byref(p))
    if nctx == 0:
        raise SageError(f"unsupported shape/flags {tuple(q.shape)} (1 <= N <= 32768, d in {{64, 128}})")
    with torch.cuda.device(dev):
        o = torch.empty_strided(q.shape, q.stride(), dtype=_out_dtype(q.dtype, fp32_out), device=dev) \
            if out is None else out
        _check_out(o, q.shape, _out_dtype(q.dtype, fp32_out), dev, "out", q.stride())
        lse = torch.empty((B, H, N), dtype=torch.float32, device=dev) if lse is None else lse
        _check_out(lse, (B, H, N), torch.float32, dev, "lse")
        ctxb = torch.empty(nctx, dtype=torch.uint8, device=dev) if ctx is None else ctx
        if ctxb.device != dev or ctxb.numel() < nctx:
            raise SageError("ctx buffer too small or on another device")
        ws = _ws.get(p, False, dev, stream) if workspace is None else workspace
        c = SageCtx(p, ctxb, (B, H, N, d), q.stride())
        _check(lib().sage_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), ctypes.byref(c.desc),
                              _ptr(ws), ws.numel(), _stream(stream, dev)), "sage_fwd")
    return o, lse, c


def backward(ctx, v, o, lse, do, dq=None, dk=None, dv=None, workspace=None, stream=None):
    """sage_bwd (Alg. 2): returns (dq, dk, dv) in the I/O dtype (fp32 with SAGE_FP32_OUT)."""
    _check_io(v, do)
    dev = do.device
    if tuple(do.shape) != tuple(ctx.shape) or ctx.buf.device != dev:
        raise SageError(f"backward: tensors {tuple(do.shape)} on {dev} do not match the forward's ctx "
                        f"{tuple(ctx.shape)} on {ctx.buf.device}")
    if (do.dtype == torch.float16) != bool(ctx.params.flags & SAGE_FP16):
        raise SageError("the backward's dtype differs from the forward's")
    B, H, N, d = ctx.shape
    st = ctx.io_stride
    _check_out(o, ctx.shape, ctx.out_dtype, dev, "o", st)
    _check_out(lse, (B, H, N), torch.float32, dev, "lse")
    v, do = _to_layout(v, st), _to_layout(do, st)  # the forward's layout (a copy only if it differs)
    if do.numel() == 0:  # the empty forward's context: empty gradients
        mk = lambda: torch.empty_strided(ctx.shape, st, dtype=ctx.out_dtype, device=dev)
        return mk(), mk(), mk()
    with torch.cuda.device(dev):
        mk = lambda: torch.empty_strided(ctx.shape, st, dtype=ctx.out_dtype, device=dev)
        dq = mk() if dq is None else dq
        dk = mk() if dk is None else dk
        dv = mk() if dv is None else dv
        for t, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
            _check_out(t, ctx.shape, ctx.out_dtype, dev, n, st)
        ws = _ws.get(ctx.params, True, dev, stream) if workspace is None else workspace
        _check(lib().sage_bwd(ctypes.byref(ctx.params), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), ctypes.byref(ctx.desc),
                              _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream(stream, dev)), "sage_bwd")
    return dq, dk, dv


def _check_gamma(g, d, device):
    if not (g.is_cuda and g.dtype == torch.float32 and g.is_contiguous() and g.shape == (d,) and g.device == device):
        raise SageError("gamma must be a contiguous CUDA fp32 [d] tensor on the inputs' device")


def forward_qknorm(xq, xk, v, gamma_q, gamma_k, eps=1e-6, causal=False, k_smooth=True, q_smooth=False,
                   softmax_scale=None, p_u8=False, out=None, lse=None, ctx=None, workspace=None, stream=None,
                   deterministic=False, p_colscale=False, fine_bwd=False):
    """sage_fwd_qknorm: QK-norm fused in front of Alg. 1.  xq, xk: the pre-norm bf16
    [B, H, N, d]; gamma_q, gamma_k: fp32 [d].  Returns (o, lse, SageCtx)."""
    _check_io(xq, xk, v)
    strides, (xq, xk, v) = _io_layout(xq, xk, v)
    B, H, N, d = xq.shape
    dev = xq.device
    _check_gamma(gamma_q, d, dev)
    _check_gamma(gamma_k, d, dev)
    p = make_params(B, H, N, d, causal, k_smooth, q_smooth, softmax_scale, p_u8, qk_norm=True,
                    deterministic=deterministic, p_colscale=p_colscale, fine_bwd=fine_bwd,
                    fp16=xq.dtype == torch.float16, strides=strides)
    if xq.numel() == 0 and d in (64, 128):  # empty batch, heads or sequence: empty results, nothing launched
        return (torch.empty_strided(xq.shape, xq.stride(), dtype=xq.dtype, device=dev),
                torch.empty((B, H, N), dtype=torch.float32, device=dev),
                SageCtx(p, torch.empty(0, dtype=torch.uint8, device=dev), (B, H, N, d), xq.stride()))
    nctx = lib().sage_ctx_bytes(ctypes.byref(p))
    if nctx == 0:
        raise SageError(f"unsupported shape/flags {tuple(xq.shape)}")
    with torch.cuda.device(dev):
        o = torch.empty_strided(xq.shape, xq.stride(), dtype=xq.dtype, device=dev) if out is None else out
        _check_out(o, xq.shape, xq.dtype, dev, "out", xq.stride())
        lse = torch.empty((B, H, N), dtype=torch.float32, device=dev) if lse is None else lse
        _check_out(lse, (B, H, N), torch.float32, dev, "lse")
        ctxb = torch.empty(nctx, dtype=torch.uint8, device=dev) if ctx is None else ctx
        if ctxb.device != dev or ctxb.numel() < nctx:
            raise SageError("ctx buffer too small or on another device")
        ws = _ws.get(p, False, dev, stream) if workspace is None else workspace
        c = SageCtx(p, ctxb, (B, H, N, d), xq.stride())
        _check(lib().sage_fwd_qknorm(ctypes.byref(p), _ptr(xq), _ptr(xk), _ptr(v), _ptr(gamma_q), _ptr(gamma_k),
                                     float(eps), _ptr(o), _ptr(lse), ctypes.byref(c.desc), _ptr(ws), ws.numel(),
                                     _stream(stream, dev)), "sage_fwd_qknorm")
    return o, lse, c


def backward_qknorm(ctx, xq, xk, gamma_q, gamma_k, v, o, lse, do, out=None, workspace=None, stream=None):
    """sage_bwd_qknorm: returns (dxq, dxk, dv, dgamma_q, dgamma_k) (into `out` if given)."""
    _check_io(xq, xk, v, o, do)
    d = xq.shape[-1]
    dev = do.device
    if tuple(do.shape) != tuple(ctx.shape) or ctx.buf.device != dev:
        raise SageError("backward_qknorm: tensors do not match the forward's ctx")
    st = ctx.io_stride
    xq, xk, v, o, do = (_to_layout(t, st) for t in (xq, xk, v, o, do))
    _check_gamma(gamma_q, d, dev)
    _check_gamma(gamma_k, d, dev)
    B, H, N, _ = ctx.shape
    _check_out(lse, (B, H, N), torch.float32, dev, "lse")
    if do.numel() == 0:  # the empty forward's context: empty dX, dV and zero dgamma
        mk = lambda: torch.empty_strided(ctx.shape, st, dtype=do.dtype, device=dev)
        return (mk(), mk(), mk(), torch.zeros(d, dtype=torch.float32, device=dev),
                torch.zeros(d, dtype=torch.float32, device=dev))
    with torch.cuda.device(dev):
        if out is None:
            mk = lambda: torch.empty_strided(ctx.shape, st, dtype=do.dtype, device=dev)
            out = (mk(), mk(), mk(), torch.empty(d, dtype=torch.float32, device=dev),
                   torch.empty(d, dtype=torch.float32, device=dev))
        dxq, dxk, dv, dgq, dgk = out
        for t, n in ((dxq, "dxq"), (dxk, "dxk"), (dv, "dv")):
            _check_out(t, ctx.shape, do.dtype, dev, n, st)
        _check_gamma(dgq, d, dev)
        _check_gamma(dgk, d, dev)
        ws = _ws.get(ctx.params, True, dev, stream) if workspace is None else workspace
        _check(lib().sage_bwd_qknorm(ctypes.byref(ctx.params), _ptr(xq), _ptr(xk), _ptr(gamma_q), _ptr(gamma_k),
                                     _ptr(v), _ptr(o), _ptr(lse), _ptr(do), ctypes.byref(ctx.desc), _ptr(dxq),
                                     _ptr(dxk), _ptr(dv), _ptr(dgq), _ptr(dgk), _ptr(ws), ws.numel(),
                                     _stream(stream, dev)), "sage_bwd_qknorm")
    return dxq, dxk, dv, dgq, dgk


class SageAttentionQKNormFn(torch.autograd.Function):
    """autograd wrapper: O = SageBwd(RMSNorm(X_q) gamma_q, RMSNorm(X_k) gamma_k, V)."""

    @staticmethod
    def forward(fctx, xq, xk, v, gamma_q, gamma_k, eps, causal, k_smooth, q_smooth, softmax_scale):
        xq, xk, v = xq.contiguous(), xk.contiguous(), v.contiguous()
        gq, gk = gamma_q.contiguous(), gamma_k.contiguous()
        o, lse, c = forward_qknorm(xq, xk, v, gq, gk, eps, causal, k_smooth, q_smooth, softmax_scale)
        fctx.sage = c
        fctx.save_for_backward(xq, xk, v, gq, gk, o, lse)
        return o

    @staticmethod
    def backward(fctx, do):
        xq, xk, v, gq, gk, o, lse = fctx.saved_tensors
        dxq, dxk, dv, dgq, dgk = backward_qknorm(fctx.sage, xq, xk, gq, gk, v, o, lse, do.contiguous())
        return dxq, dxk, dv, dgq, dgk, None, None, None, None, None


def sage_attention_qknorm(xq, xk, v, gamma_q, gamma_k, eps=1e-6, causal=False, k_smooth=True, q_smooth=False,
                          softmax_scale=None):
    return SageAttentionQKNormFn.apply(xq, xk, v, gamma_q, gamma_k, eps, causal, k_smooth, q_smooth, softmax_scale)


class SageAttentionFn(torch.autograd.Function):
    """autograd wrapper: O = SageBwd(Q, K, V) with the INT8 backward of Alg. 2."""

    @staticmethod
    def forward(fctx, q, k, v, causal, k_smooth, q_smooth, softmax_scale):
        o, lse, c = forward(q, k, v, causal, k_smooth, q_smooth, softmax_scale)
        fctx.sage = c
        fctx.save_for_backward(v, o, lse)
        return o

    @staticmethod
    def backward(fctx, do):
        v, o, lse = fctx.saved_tensors
        dq, dk, dv = backward(fctx.sage, v, o, lse, do)
        return dq, dk, dv, None, None, None, None


def sage_attention(q, k, v, causal=False, k_smooth=True, q_smooth=False, softmax_scale=None):
    return SageAttentionFn.apply(q, k, v, causal, k_smooth, q_smooth, softmax_scale)


def debug_umma(mode, a, b, K=None, N=None):
    """One UMMA tile through the kernels' descriptor code (include/sage.h sage_debug_umma)."""
    if mode in (0, 3, 5):
        K = a.shape[1]
        N = 128
        out = torch.empty((128, 128), dtype=torch.int32 if mode == 0 else torch.float32, device=a.device)
    else:
        K = 128
        N = b.shape[1]
        out = torch.empty((128, N), dtype=torch.int32, device=a.device)
    _check(lib().sage_debug_umma(mode, K, N, _ptr(a), _ptr(b), _ptr(out), _stream(None)), "sage_debug_umma")
    return out


def debug_dump(heads, N, device, d=None, acc=False):
    """Arm sage_debug_dump (libsage_trace.so only) for heads [0, heads) of sequence length N:
    returns the device buffers every later sage_bwd fills (include/sage.h); heads=0 disarms.
    acc=True (head dim d) also arms sage_debug_dump_acc: the int32 S^T, dV, dK, dQ tile accumulators and the
    fp32 dP^T."""
    if heads == 0:
        _check(lib().sage_debug_dump(None, None, None, None, None, 0), "sage_debug_dump")
        _check(lib().sage_debug_dump_acc(None, None, None, None, None), "sage_debug_dump_acc")
        return None
    if N % 128:
        raise SageError("the tile dumps need N % 128 == 0")
    T = N // 128
    bufs = dict(p_hat_t=torch.zeros((heads, N, N), dtype=torch.int8, device=device),
                s_p=torch.zeros((heads, T, T), dtype=torch.float32, device=device),
                ds_hat_t=torch.zeros((heads, N, N), dtype=torch.int8, device=device),
                s_ds=torch.zeros((heads, T, T), dtype=torch.float32, device=device),
                ds_t=torch.zeros((heads, N, N), dtype=torch.float32, device=device))
    _check(lib().sage_debug_dump(_ptr(bufs["p_hat_t"]), _ptr(bufs["s_p"]), _ptr(bufs["ds_hat_t"]),
                                 _ptr(bufs["s_ds"]), _ptr(bufs["ds_t"]), heads), "sage_debug_dump")
    if acc:
        bufs.update(s_t=torch.zeros((heads, N, N), dtype=torch.int32, device=device),
                    dv_t=torch.zeros((heads, T, N, d), dtype=torch.int32, device=device),
                    dk_t=torch.zeros((heads, T, N, d), dtype=torch.int32, device=device),
                    dq_t=torch.zeros((heads, T, N, d), dtype=torch.int32, device=device),
                    dp_t=torch.zeros((heads, N, N), dtype=torch.float32, device=device))
        _check(lib().sage_debug_dump_acc(_ptr(bufs["s_t"]), _ptr(bufs["dv_t"]), _ptr(bufs["dk_t"]),
                                         _ptr(bufs["dq_t"]), _ptr(bufs["dp_t"])), "sage_debug_dump_acc")
    else:
        _check(lib().sage_debug_dump_acc(None, None, None, None, None), "sage_debug_dump_acc")
    return bufs


def debug_fwd_dump(heads, N, d, device):
    """Arm sage_debug_fwd_dump (libsage_trace.so only): every later sage_fwd writes K2's int32 S, P^,
    s_P and int32 PV accumulators of heads [0, heads) into the returned buffers; heads=0 disarms."""
    if heads == 0:
        _check(lib().sage_debug_fwd_dump(None, None, None, None, 0), "sage_debug_fwd_dump")
        return None
    if N % 128:
        raise SageError("the tile dumps need N % 128 == 0")
    T = N // 128
    bufs = dict(s=torch.zeros((heads, N, N), dtype=torch.int32, device=device),
                p_hat=torch.zeros((heads, N, N), dtype=torch.uint8, device=device),
                s_p=torch.zeros((heads, N, T), dtype=torch.float32, device=device),
                pv=torch.zeros((heads, T, N, d), dtype=torch.int32, device=device))
    _check(lib().sage_debug_fwd_dump(_ptr(bufs["s"]), _ptr(bufs["p_hat"]), _ptr(bufs["s_p"]), _ptr(bufs["pv"]), heads),
           "sage_debug_fwd_dump")
    return bufs


def profile_enable(on=True):
    """Record events around the fused kernels K2/K4 and count launches (sage_profile_enable)."""
    _check(lib().sage_profile_enable(int(on)), "sage_profile_enable")


def profile_read():
    """-> dict(fwd_ms, bwd_ms, n_fwd, n_bwd, launches) since the last read (sage_profile_read)."""
    f, b = ctypes.c_double(), ctypes.c_double()
    nf, nb, nl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().sage_profile_read(ctypes.byref(f), ctypes.byref(b), ctypes.byref(nf), ctypes.byref(nb),
                                   ctypes.byref(nl)), "sage_profile_read")
    return dict(fwd_ms=f.value, bwd_ms=b.value, n_fwd=nf.value, n_bwd=nb.value, launches=nl.value)


def default_scale(d):
    return 1.0 / math.sqrt(d)
