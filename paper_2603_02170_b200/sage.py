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
SAGE_FINE_BWD, SAGE_FP16 = 128, 256
_STATUS = {0: "SAGE_OK", 1: "SAGE_ERR_INVALID_VALUE", 2: "SAGE_ERR_UNSUPPORTED", 3: "SAGE_ERR_MISALIGNED",
           4: "SAGE_ERR_WORKSPACE", 5: "SAGE_ERR_CUDA", 6: "SAGE_ERR_ARCH"}

# exported symbols of include/sage.h
SYMBOLS = ("sage_ctx_bytes", "sage_workspace_bytes", "sage_fwd", "sage_bwd", "sage_fwd_qknorm", "sage_bwd_qknorm",
           "sage_ctx_get_view",
           "sage_ws_get_view", "sage_debug_umma", "sage_debug_trace", "sage_debug_dump", "sage_profile_enable", "sage_profile_read",
           "sage_status_string", "sage_last_cuda_error", "sage_version")


class SageParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("heads", ctypes.c_int32), ("seqlen", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("flags", ctypes.c_uint32), ("softmax_scale", ctypes.c_float)]


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
        L.sage_fwd.argtypes = [pp, P, P, P, P, P, P, S, P, S, P]
        L.sage_bwd.argtypes = [pp, P, P, P, P, P, S, P, P, P, P, S, P]
        L.sage_fwd_qknorm.argtypes = [pp, P, P, P, P, P, ctypes.c_float, P, P, P, S, P, S, P]
        L.sage_bwd_qknorm.argtypes = [pp, P, P, P, P, P, P, P, P, P, S, P, P, P, P, P, P, S, P]
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
                p_u8=False, qk_norm=False, deterministic=False, p_colscale=False, fine_bwd=False, fp16=False):
    flags = (SAGE_CAUSAL if causal else 0) | (SAGE_K_SMOOTH if k_smooth else 0) | (SAGE_Q_SMOOTH if q_smooth else 0) | \
        (SAGE_P_U8 if p_u8 else 0) | (SAGE_QK_NORM if qk_norm else 0) | (SAGE_DETERMINISTIC if deterministic else 0) | \
        (SAGE_P_COLSCALE if p_colscale else 0) | (SAGE_FINE_BWD if fine_bwd else 0) | (SAGE_FP16 if fp16 else 0)
    return SageParams(batch, heads, seqlen, head_dim, flags, 0.0 if softmax_scale is None else softmax_scale)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_io(*ts):
    """All tensors contiguous CUDA [B, H, N, d] of one I/O dtype: bf16, or fp16 (SAGE_FP16)."""
    ref = ts[0]
    for t in ts:
        if not (t.is_cuda and t.dtype in (torch.bfloat16, torch.float16) and t.is_contiguous() and t.dim() == 4):
            raise SageError("tensors must be contiguous CUDA bf16 or fp16 [B, H, N, d]")
        if t.shape != ref.shape or t.device != ref.device or t.dtype != ref.dtype:
            raise SageError("shape/device/dtype mismatch")


class SageCtx:
    """Forward->backward state (Alg. 2 inputs): the caller-owned ctx buffer plus params."""

    def __init__(self, params, ctx, shape):
        self.params, self.buf, self.shape = params, ctx, shape

    def view(self):
        """Device tensors of the context (Q^, K^, scales, mu_K, mu_Q, bias) -- no copies."""
        v = SageCtxView()
        _check(lib().sage_ctx_get_view(ctypes.byref(self.params), _ptr(self.buf), ctypes.byref(v)), "ctx_view")
        B, H, N, d = self.shape
        T = N // 128
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
    """Reusable scratch buffers (sage_workspace_bytes), grown on demand per device."""

    def __init__(self):
        self.bufs = {}

    def get(self, params, backward, device):
        n = lib().sage_workspace_bytes(ctypes.byref(params), int(backward))
        if n == 0:
            raise SageError("invalid sage_params")
        device = torch.device(device)
        if device.index is None:
            device = torch.device(device.type, torch.cuda.current_device())
        key = (str(device), backward)
        b = self.bufs.get(key)
        if b is None or b.numel() < n:
            b = torch.empty(n, dtype=torch.uint8, device=device)
            self.bufs[key] = b
        return b


_ws = Workspace()


def ws_view(params, backward, ws):
    v = SageWsView()
    _check(lib().sage_ws_get_view(ctypes.byref(params), int(backward), _ptr(ws), ctypes.byref(v)), "ws_view")
    return v


def forward(q, k, v, causal=False, k_smooth=True, q_smooth=False, softmax_scale=None, out=None, lse=None,
            ctx=None, workspace=None, stream=None, p_u8=False, deterministic=False, p_colscale=False,
            fine_bwd=False):
    """sage_fwd (Alg. 1): returns (o, lse, SageCtx).  q, k, v: CUDA bf16 [B, H, N, d].
    p_u8: the unsigned-P^ variant (SAGE_P_U8); deterministic: a bitwise reproducible backward
    (SAGE_DETERMINISTIC); p_colscale: per-key psi(P) in the backward (SAGE_P_COLSCALE); fine_bwd: per-key
    psi(P) and per-key / per-query psi(dS) (SAGE_FINE_BWD).  The backward inherits them through the ctx."""
    _check_io(q, k, v)
    B, H, N, d = q.shape
    p = make_params(B, H, N, d, causal, k_smooth, q_smooth, softmax_scale, p_u8, deterministic=deterministic,
                    p_colscale=p_colscale, fine_bwd=fine_bwd, fp16=q.dtype == torch.float16)
    nctx = lib().sage_ctx_bytes(ctypes.byref(p))
    if nctx == 0:
        raise SageError(f"unsupported shape/flags {tuple(q.shape)} (N % 128 == 0, d in {{64, 128}})")
    o = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, H, N), dtype=torch.float32, device=q.device) if lse is None else lse
    ctxb = torch.empty(nctx, dtype=torch.uint8, device=q.device) if ctx is None else ctx
    ws = _ws.get(p, False, q.device) if workspace is None else workspace
    _check(lib().sage_fwd(ctypes.byref(p), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(ctxb), ctxb.numel(),
                          _ptr(ws), ws.numel(), _stream(stream)), "sage_fwd")
    return o, lse, SageCtx(p, ctxb, (B, H, N, d))


def backward(ctx, v, o, lse, do, dq=None, dk=None, dv=None, workspace=None, stream=None):
    """sage_bwd (Alg. 2): returns (dq, dk, dv) in the I/O dtype."""
    _check_io(v, o, do)
    if (do.dtype == torch.float16) != bool(ctx.params.flags & SAGE_FP16):
        raise SageError("the backward's dtype differs from the forward's")
    dq = torch.empty_like(do) if dq is None else dq
    dk = torch.empty_like(do) if dk is None else dk
    dv = torch.empty_like(do) if dv is None else dv
    ws = _ws.get(ctx.params, True, do.device) if workspace is None else workspace
    _check(lib().sage_bwd(ctypes.byref(ctx.params), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), _ptr(ctx.buf),
                          ctx.buf.numel(), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream(stream)),
           "sage_bwd")
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
    B, H, N, d = xq.shape
    _check_gamma(gamma_q, d, xq.device)
    _check_gamma(gamma_k, d, xq.device)
    p = make_params(B, H, N, d, causal, k_smooth, q_smooth, softmax_scale, p_u8, qk_norm=True,
                    deterministic=deterministic, p_colscale=p_colscale, fine_bwd=fine_bwd,
                    fp16=xq.dtype == torch.float16)
    nctx = lib().sage_ctx_bytes(ctypes.byref(p))
    if nctx == 0:
        raise SageError(f"unsupported shape/flags {tuple(xq.shape)}")
    o = torch.empty_like(xq) if out is None else out
    lse = torch.empty((B, H, N), dtype=torch.float32, device=xq.device) if lse is None else lse
    ctxb = torch.empty(nctx, dtype=torch.uint8, device=xq.device) if ctx is None else ctx
    ws = _ws.get(p, False, xq.device) if workspace is None else workspace
    _check(lib().sage_fwd_qknorm(ctypes.byref(p), _ptr(xq), _ptr(xk), _ptr(v), _ptr(gamma_q), _ptr(gamma_k),
                                 float(eps), _ptr(o), _ptr(lse), _ptr(ctxb), ctxb.numel(), _ptr(ws), ws.numel(),
                                 _stream(stream)), "sage_fwd_qknorm")
    return o, lse, SageCtx(p, ctxb, (B, H, N, d))


def backward_qknorm(ctx, xq, xk, gamma_q, gamma_k, v, o, lse, do, out=None, workspace=None, stream=None):
    """sage_bwd_qknorm: returns (dxq, dxk, dv, dgamma_q, dgamma_k) (into `out` if given)."""
    _check_io(xq, xk, v, o, do)
    d = xq.shape[-1]
    _check_gamma(gamma_q, d, xq.device)
    _check_gamma(gamma_k, d, xq.device)
    if out is None:
        out = (torch.empty_like(do), torch.empty_like(do), torch.empty_like(do),
               torch.empty(d, dtype=torch.float32, device=do.device),
               torch.empty(d, dtype=torch.float32, device=do.device))
    dxq, dxk, dv, dgq, dgk = out
    ws = _ws.get(ctx.params, True, do.device) if workspace is None else workspace
    _check(lib().sage_bwd_qknorm(ctypes.byref(ctx.params), _ptr(xq), _ptr(xk), _ptr(gamma_q), _ptr(gamma_k), _ptr(v),
                                 _ptr(o), _ptr(lse), _ptr(do), _ptr(ctx.buf), ctx.buf.numel(), _ptr(dxq), _ptr(dxk),
                                 _ptr(dv), _ptr(dgq), _ptr(dgk), _ptr(ws), ws.numel(), _stream(stream)),
           "sage_bwd_qknorm")
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
        o, lse, c = forward(q.contiguous(), k.contiguous(), v.contiguous(), causal, k_smooth, q_smooth,
                            softmax_scale)
        fctx.sage = c
        fctx.save_for_backward(v, o, lse)
        return o

    @staticmethod
    def backward(fctx, do):
        v, o, lse = fctx.saved_tensors
        dq, dk, dv = backward(fctx.sage, v, o, lse, do.contiguous())
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


def debug_dump(heads, N, device):
    """Arm sage_debug_dump (libsage_trace.so only) for heads [0, heads) of sequence length N:
    returns the device buffers every later sage_bwd fills (include/sage.h); heads=0 disarms."""
    if heads == 0:
        _check(lib().sage_debug_dump(None, None, None, None, None, 0), "sage_debug_dump")
        return None
    T = N // 128
    bufs = dict(p_hat_t=torch.zeros((heads, N, N), dtype=torch.int8, device=device),
                s_p=torch.zeros((heads, T, T), dtype=torch.float32, device=device),
                ds_hat_t=torch.zeros((heads, N, N), dtype=torch.int8, device=device),
                s_ds=torch.zeros((heads, T, T), dtype=torch.float32, device=device),
                ds_t=torch.zeros((heads, N, N), dtype=torch.float32, device=device))
    _check(lib().sage_debug_dump(_ptr(bufs["p_hat_t"]), _ptr(bufs["s_p"]), _ptr(bufs["ds_hat_t"]),
                                 _ptr(bufs["s_ds"]), _ptr(bufs["ds_t"]), heads), "sage_debug_dump")
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
