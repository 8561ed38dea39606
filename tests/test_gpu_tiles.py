"""Tier A / B / C parity of the FUSED kernels' own intermediates (SURVEY.md 8(c) parity contract).

libsage_trace.so's dumps (sage_debug_fwd_dump, sage_debug_dump + sage_debug_dump_acc; include/sage.h)
write, with the production kernel code, the int32 tile accumulators and int8 operands K2 and K4 form:

- Tier A (bit-exact from the inputs alone): K2's S = Q^_i K^_j^T of every processed tile (Alg. 1 line 7,
  P:655) equals the exact integer product of the oracle's Q^, K^; K4's recomputed S^T (Alg. 2 line 5)
  is the same tile, bit for bit.
- Tier B (bit-exact given the dumped int8 operands): K2's P^ V^_j (Alg. 1 line 10), K4's P^^T dO^_i
  (dV, line 7), dS^^T Q^_i (dK, line 11) and dS^ K^_j (dQ, line 10) accumulators equal the dumped operands
  re-multiplied in int64 -- this checks the fused kernels' descriptors, swizzles, stage offsets and TMEM
  column placements, not a stand-alone test kernel's.  K4's BF16 dP^T (line 8) equals dO_i V_j^T within
  fp32 accumulation (1e-6 of the sum of |products|).
- Tier C (statistical, exp-bit dependent): K2's per-token P^ and s_P (Alg. 1 line 9) against the
  oracle's: >= 99.99% of P^ identical, none more than 1 LSB apart, s_P within 64 fp32 ulp.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_02170_b200 import build, sage
from paper_2603_02170_b200.inputs import make_inputs
from tests.metrics import f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def trace_lib():
    assert torch.cuda.is_available() and torch.cuda.get_device_capability() == (10, 0)
    if not __import__("os").path.exists(build.TRACE_LIB):
        build.build(trace=True)
    oracle.build()
    old = sage.use_library(build.TRACE_LIB)
    yield
    sage.debug_dump(0, 0, None)
    sage.debug_fwd_dump(0, 0, 0, None)
    sage.use_library(old)


CASES = [
    # (B, H, N, d, causal, k_smooth, q_smooth, recipe, p_u8)
    (1, 2, 384, 64, True, True, False, "qknorm", False),
    (1, 2, 256, 64, False, True, False, "gauss", False),
    (1, 2, 384, 128, True, True, True, "outlier_kq", False),
    (1, 2, 256, 128, False, True, False, "qknorm", False),
    (2, 1, 384, 128, True, False, False, "gauss", False),
    (1, 2, 384, 64, True, True, False, "qknorm", True),
]


def _ws_tensor(ws, addr, n, dtype, shape):
    off = addr - ws.data_ptr()
    nbytes = n * torch.empty((), dtype=dtype).element_size()
    return ws[off:off + nbytes].view(dtype).view(shape).cpu().numpy()


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe,u8", CASES)
def test_fused_tiles(trace_lib, B, H, N, d, causal, ks, qs, recipe, u8):
    BH, T = B * H, N // 128
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=1100 + N + d)
    dev = torch.device("cuda")
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    fb = sage.debug_fwd_dump(BH, N, d, dev)
    bb = sage.debug_dump(BH, N, dev, d=d, acc=True)
    o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, k_smooth=ks, q_smooth=qs, p_u8=u8)
    sage.backward(ctx, vd, o, lse, dod)
    torch.cuda.synchronize()
    sage.debug_fwd_dump(0, 0, 0, None)
    sage.debug_dump(0, 0, None)
    fb = {n: t.cpu().numpy() for n, t in fb.items()}
    bb = {n: t.cpu().numpy() for n, t in bb.items()}

    # Tier-A operands: the GPU's own Q^, K^ (ctx), V^ (forward workspace), dO^ (backward workspace)
    view = ctx.view()
    q8 = view["q_i8"].cpu().numpy().reshape(BH, N, d).astype(np.int64)
    k8 = view["k_i8"].cpu().numpy().reshape(BH, N, d).astype(np.int64)
    wsf = sage._ws.get(ctx.params, False, dev)
    v8 = _ws_tensor(wsf, sage.ws_view(ctx.params, False, wsf).v_i8, BH * N * d, torch.int8, (BH, N, d)).astype(np.int64)
    wsb = sage._ws.get(ctx.params, True, dev)
    do8 = _ws_tensor(wsb, sage.ws_view(ctx.params, True, wsb).do_i8, BH * N * d, torch.int8, (BH, N, d)).astype(np.int64)
    kw = dict(causal=causal, k_smooth=ks, q_smooth=qs, p_u8=u8)
    f = oracle.fwd(*(f64(t).reshape(BH, N, d) for t in (q, k, v)), tiles=True, **kw)
    np.testing.assert_array_equal(q8, f["q8"])
    np.testing.assert_array_equal(k8, f["k8"])
    np.testing.assert_array_equal(v8, f["v8"])

    pdt = np.uint8 if u8 else np.int8
    dof, vf = (f64(t).reshape(BH, N, d) for t in (do, v))
    blk = lambda t: slice(t * 128, (t + 1) * 128)
    tiles = [(i, j) for i in range(T) for j in range(T) if not causal or j <= i]
    n_p = n_same = 0
    max_p_diff = 0
    sp_ulp = 0.0
    for h in range(BH):
        s_ref = q8[h] @ k8[h].T                        # exact; |S| <= d 127^2 < 2^31
        p_t = bb["p_hat_t"][h].view(pdt).astype(np.int64)   # [N kv][N q]
        ds_t = bb["ds_hat_t"][h].astype(np.int64)
        for i, j in tiles:
            I, J = blk(i), blk(j)
            # Tier A: forward S and the backward's recomputed S^T, against the exact product
            np.testing.assert_array_equal(fb["s"][h][I, J], s_ref[I, J], err_msg=f"K2 S h{h} ({i},{j})")
            np.testing.assert_array_equal(bb["s_t"][h][J, I].T, s_ref[I, J], err_msg=f"K4 S^T h{h} ({i},{j})")
            # Tier B: K2's PV accumulator = its own P^ times V^_j
            p_fwd = fb["p_hat"][h][I, J].astype(np.int64)
            np.testing.assert_array_equal(fb["pv"][h, j, I], p_fwd @ v8[h][J], err_msg=f"K2 PV h{h} ({i},{j})")
            # Tier B: K4's dV, dK, dQ accumulators = the dumped P^^T / dS^^T times dO^_i, Q^_i, K^_j
            np.testing.assert_array_equal(bb["dv_t"][h, i, J], p_t[J, I] @ do8[h][I], err_msg=f"K4 dV h{h} ({i},{j})")
            np.testing.assert_array_equal(bb["dk_t"][h, i, J], ds_t[J, I] @ q8[h][I], err_msg=f"K4 dK h{h} ({i},{j})")
            np.testing.assert_array_equal(bb["dq_t"][h, j, I], ds_t[J, I].T @ k8[h][J], err_msg=f"K4 dQ h{h} ({i},{j})")
            # the BF16 dP MMA (line 8): exact products of the I/O values, fp32 accumulation of d terms
            dp_ref = dof[h][I] @ vf[h][J].T
            bound = 1e-6 * (np.abs(dof[h][I]) @ np.abs(vf[h][J]).T) + 1e-30
            assert (np.abs(bb["dp_t"][h][J, I].T - dp_ref) <= bound).all(), f"K4 dP h{h} ({i},{j})"
            # Tier C: the forward's per-token P^ and s_P against the oracle's
            ref_p = f["p8"][h][I, J].astype(np.int64)
            diff = np.abs(p_fwd - ref_p)
            n_p += diff.size
            n_same += int((diff == 0).sum())
            max_p_diff = max(max_p_diff, int(diff.max()))
            sp_g = fb["s_p"][h][I, j].astype(np.float64)
            sp_r = f["sp"][h][I, j]
            ulp = np.spacing(sp_r.astype(np.float32)).astype(np.float64)
            sp_ulp = max(sp_ulp, float((np.abs(sp_g - sp_r) / ulp).max()))
    assert max_p_diff <= 1 and n_same / n_p >= 0.9999, (max_p_diff, n_same / n_p)
    assert sp_ulp <= 64, sp_ulp


@pytest.mark.parametrize("d,causal", [(64, True), (128, False)])
def test_fused_tiles_pv_fp8(trace_lib, d, causal):
    """SAGE_PV_FP8 (Tier B on the fused kernel): K2's fp32 P^V^ accumulator (kind::f8f6f4) equals its own
    dumped E4M3 P^ times the E4M3 V^ within fp32 accumulation (1e-6 of the sum of |products|); every dumped
    P^ is a finite E4M3 value in [0, 448] with 448 attained in every processed row (the row max)."""
    B, H, N = 1, 2, 384
    BH, T = B * H, N // 128
    q, k, v, do = make_inputs(B, H, N, d, "qknorm", seed=1500 + d)
    dev = torch.device("cuda")
    qd, kd, vd = (t.to(dev) for t in (q, k, v))
    fb = sage.debug_fwd_dump(BH, N, d, dev)
    o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, pv_fp8=True)
    torch.cuda.synchronize()
    sage.debug_fwd_dump(0, 0, 0, None)
    wsf = sage._ws.get(ctx.params, False, dev)
    v8 = _ws_tensor(wsf, sage.ws_view(ctx.params, False, wsf).v_i8, BH * N * d, torch.int8, (BH, N, d))
    v8 = torch.from_numpy(v8).view(torch.float8_e4m3fn).double().numpy()
    p8 = fb["p_hat"].cpu().view(torch.float8_e4m3fn).double().numpy()
    pv = fb["pv"].cpu().view(torch.float32).double().numpy()
    blk = lambda t: slice(t * 128, (t + 1) * 128)
    same = total = 0
    for h in range(BH):
        for i in range(T):
            for j in range(T):
                if causal and j > i:
                    continue
                P, V = p8[h][blk(i), blk(j)], v8[h][blk(j)]
                ref = P @ V
                bound = 1e-6 * (np.abs(P) @ np.abs(V)) + 1e-30
                assert (np.abs(pv[h, j, blk(i)] - ref) <= bound).all(), (h, i, j)
                assert np.isfinite(P).all() and P.min() >= 0 and (P.max(axis=1) == 448.0).all(), (h, i, j)
