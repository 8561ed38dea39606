"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tier A (bit-exact): mu_K, mu_Q, Q^, K^, V^, dO^ and their fp32 scales.
Tier B (bit-exact): int32 UMMA tiles for every operand configuration the kernels use.
Outputs O, dQ, dK, dV: rel-L2 <= 2e-3 and cos >= 0.9999 against the quantised oracle,
both sides rounded to bf16 (BASELINE.json north_star tolerance; reading A18).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_02170_b200 import sage
from paper_2603_02170_b200.inputs import CONFIGS, make_inputs
from tests.metrics import cos_sim, f64, rel_l2, round_bf16, round_fp16

pytestmark = pytest.mark.gpu

REL_TOL, COS_TOL = 2e-3, 0.9999


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available(), "gpu tests need an sm_100 device"
    assert torch.cuda.get_device_capability() == (10, 0), torch.cuda.get_device_capability()
    sage.lib()
    oracle.build()


def _run(q, k, v, do, causal, k_smooth, q_smooth, p_u8=False, deterministic=False, p_colscale=False,
         fine_bwd=False, softmax_scale=None, fp32_out=False):
    dev = "cuda"
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, k_smooth=k_smooth, q_smooth=q_smooth, p_u8=p_u8,
                               deterministic=deterministic, p_colscale=p_colscale, fine_bwd=fine_bwd,
                               softmax_scale=softmax_scale, fp32_out=fp32_out)
    dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
    torch.cuda.synchronize()
    return dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv, ctx=ctx)


def _oracle(q, k, v, do, heads, causal, k_smooth, q_smooth, p_u8=False, p_col=False, ds_fine=False, tau=None,
            o_round=round_bf16):
    """Oracle on the selected flattened heads; O is stored as bf16 before the backward (A15)."""
    B, H, N, d = q.shape
    sel = lambda t: f64(t).reshape(B * H, N, d)[heads]
    qn, kn, vn, don = map(sel, (q, k, v, do))
    kw = dict(causal=causal, k_smooth=k_smooth, q_smooth=q_smooth, p_u8=p_u8, tau=tau)
    f = oracle.fwd(qn, kn, vn, **kw)
    o_st = o_round(f["o"])
    b = oracle.bwd(qn, kn, vn, o_st, don, f["lse"], p_col=p_col, ds_fine=ds_fine, **kw)
    return f, b


def _compare(gpu, f, b, heads, B, H, N, d, out_round=round_bf16):
    """rel-L2 / cos over all compared heads (global flatten, A21) and the worst single head; max |dL|."""
    flat = lambda t: f64(t).reshape(B * H, N, d)[heads]
    res = {}
    for name, ref in (("o", f["o"]), ("dq", b["dq"]), ("dk", b["dk"]), ("dv", b["dv"])):
        got = flat(gpu[name])
        ref = out_round(ref)
        worst = max(rel_l2(ref[h], got[h]) for h in range(len(heads)))
        res[name] = (rel_l2(ref, got), cos_sim(ref, got), worst)
    lse = f64(gpu["lse"]).reshape(B * H, N)[heads]
    res["lse"] = float(np.abs(lse - f["lse"]).max())
    return res


def _assert_ok(res, what):
    """North-star tolerance: rel-L2 <= 2e-3 and cos >= 0.9999 globally and for every head; L within 1e-5
    absolute."""
    for name in ("o", "dq", "dk", "dv"):
        rl, cs, worst = res[name]
        assert rl <= REL_TOL and cs >= COS_TOL and worst <= REL_TOL, (what, name, rl, cs, worst, res)
    assert res["lse"] <= 1e-5, (what, res)


# ------------------------------------------------------------------ Tier B: UMMA tiles
@pytest.mark.parametrize("K", [64, 128])
def test_umma_s_tile_kmajor(K):
    g = torch.Generator().manual_seed(K)
    a = torch.randint(-127, 128, (128, K), generator=g, dtype=torch.int8)
    b = torch.randint(-127, 128, (128, K), generator=g, dtype=torch.int8)
    d = sage.debug_umma(0, a.cuda(), b.cuda()).cpu().numpy()
    np.testing.assert_array_equal(d, a.numpy().astype(np.int64) @ b.numpy().astype(np.int64).T)


@pytest.mark.parametrize("mode", [1, 2, 4, 6, 7])
@pytest.mark.parametrize("N", [64, 128])
def test_umma_mn_major(mode, N):
    """modes 1 / 4: A K-major from smem / from TMEM (TS); mode 2: A MN-major (dQ);
    modes 6 / 7: as 1 / 4 with an unsigned u8 A (SAGE_P_U8: P^ in [0, 255])."""
    g = torch.Generator().manual_seed(10 * mode + N)
    if mode >= 6:
        a = torch.randint(0, 256, (128, 128), generator=g, dtype=torch.uint8)
    else:
        lo = 0 if mode == 1 else -127      # mode 1 is the P^ path (values in [0, 127])
        a = torch.randint(lo, 128, (128, 128), generator=g, dtype=torch.int8)
    b = torch.randint(-127, 128, (128, N), generator=g, dtype=torch.int8)
    d = sage.debug_umma(mode, a.cuda(), b.cuda()).cpu().numpy()
    A = a.numpy().astype(np.int64)
    if mode == 2:                           # a holds A^T ([K][M], the dS^^T tile)
        A = A.T
    np.testing.assert_array_equal(d, A @ b.numpy().astype(np.int64))


@pytest.mark.parametrize("mode", [3, 5])
@pytest.mark.parametrize("K", [64, 128])
def test_umma_bf16_dp_tile(mode, K):
    """mode 3: both bf16 operands from smem; mode 5: A (V_j) from TMEM."""
    g = torch.Generator().manual_seed(K + 1)
    a = torch.randn(128, K, generator=g).to(torch.bfloat16)
    b = torch.randn(128, K, generator=g).to(torch.bfloat16)
    d = sage.debug_umma(mode, a.cuda(), b.cuda()).cpu().numpy()
    ref = f64(a) @ f64(b).T
    assert np.abs(d - ref).max() <= 1e-4 * np.abs(ref).max()


# ------------------------------------------------------------------ Tier A: quantised inputs
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("q_smooth", [False, True])
def test_tier_a_bit_exact(d, q_smooth):
    B, H, N = 1, 2, 384
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=21 + d)
    gpu = _run(q, k, v, do, True, True, q_smooth)
    view = gpu["ctx"].view()
    f, b = _oracle(q, k, v, do, list(range(B * H)), True, True, q_smooth)
    T = N // 128
    np.testing.assert_array_equal(view["mu_k"].cpu().numpy().reshape(B * H, d), f["mu_k"])
    np.testing.assert_array_equal(view["q_i8"].cpu().numpy().reshape(B * H, N, d), f["q8"])
    np.testing.assert_array_equal(view["k_i8"].cpu().numpy().reshape(B * H, N, d), f["k8"])
    np.testing.assert_array_equal(view["q_scale"].cpu().numpy().reshape(B * H, T), f["sq"])
    np.testing.assert_array_equal(view["k_scale"].cpu().numpy().reshape(B * H, T), f["sk"])
    if q_smooth:
        np.testing.assert_array_equal(view["mu_q"].cpu().numpy().reshape(B * H, T, d), f["mu_q"])
        bias = view["bias"].cpu().numpy().reshape(B * H, T, N).astype(np.float64)
        assert np.abs(bias - f["bias"]).max() <= 1e-5 * np.abs(f["bias"]).max()
    # V^ and dO^ live in the workspaces
    p = gpu["ctx"].params
    wsf = sage._ws.get(p, False, torch.device("cuda"))
    wv = sage.ws_view(p, False, wsf)
    base = wsf.data_ptr()
    v8 = wsf[wv.v_i8 - base: wv.v_i8 - base + B * H * N * d].view(torch.int8).cpu().numpy()
    sv = wsf[wv.v_scale - base: wv.v_scale - base + B * H * T * 4].view(torch.float32).cpu().numpy()
    np.testing.assert_array_equal(v8.reshape(B * H, N, d), f["v8"])
    np.testing.assert_array_equal(sv.reshape(B * H, T), f["sv"])
    wsb = sage._ws.get(p, True, torch.device("cuda"))
    wb = sage.ws_view(p, True, wsb)
    base = wsb.data_ptr()
    do8 = wsb[wb.do_i8 - base: wb.do_i8 - base + B * H * N * d].view(torch.int8).cpu().numpy()
    sdo = wsb[wb.do_scale - base: wb.do_scale - base + B * H * T * 4].view(torch.float32).cpu().numpy()
    np.testing.assert_array_equal(do8.reshape(B * H, N, d), b["do8"])
    np.testing.assert_array_equal(sdo.reshape(B * H, T), b["sdo"])
    delta = wsb[wb.delta - base: wb.delta - base + B * H * N * 4].view(torch.float32).cpu().numpy()
    # delta = rowsum(dO o O) from the O the forward stored (A15): the oracle given the GPU's stored O
    # (exact fp64 sum of exact products) rounded once to fp32 -- bit-exact
    flat = lambda t: f64(t).reshape(B * H, N, d)
    b_st = oracle.bwd(flat(q), flat(k), flat(v), flat(gpu["o"]), flat(do), f["lse"], causal=True, k_smooth=True,
                      q_smooth=q_smooth)
    np.testing.assert_array_equal(delta.reshape(B * H, N), b_st["delta"].astype(np.float32))


# ------------------------------------------------------------------ fused fwd + bwd parity
SMALL = [
    # (B, H, N, d, causal, k_smooth, q_smooth, recipe)
    (1, 2, 128, 64, True, True, False, "outlier_k"),      # C1 (BASELINE.json configs[0])
    (1, 2, 128, 64, True, True, False, "gauss"),
    (1, 2, 256, 64, False, True, False, "qknorm"),
    (1, 2, 384, 64, True, True, False, "qknorm"),
    (1, 2, 512, 128, True, True, False, "qknorm"),
    (1, 2, 384, 128, False, True, False, "outlier_k"),
    (1, 2, 384, 128, True, False, False, "gauss"),
    (1, 2, 512, 64, True, True, True, "outlier_kq"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
    (2, 1, 256, 128, False, True, True, "outlier_kq"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", SMALL)
def test_fwd_bwd_parity_small(B, H, N, d, causal, ks, qs, recipe):
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=100 + N + d)
    gpu = _run(q, k, v, do, causal, ks, qs)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, ks, qs)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), (B, H, N, d, causal, ks, qs, recipe))


P_U8_CASES = [
    (1, 2, 384, 64, True, True, False, "qknorm"),
    (1, 2, 256, 64, False, True, False, "gauss"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
    (1, 2, 256, 128, False, True, False, "qknorm"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", P_U8_CASES)
def test_fwd_bwd_parity_p_u8(B, H, N, d, causal, ks, qs, recipe):
    """SAGE_P_U8 (P^ in 0..255, u8 x s8 PV / dV MMAs) against the oracle's ORC_P_U8 mode."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=200 + N + d)
    gpu = _run(q, k, v, do, causal, ks, qs, p_u8=True)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, ks, qs, p_u8=True)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), (B, H, N, d, causal, ks, qs, recipe, "u8"))


PCOL_CASES = [
    (1, 2, 384, 64, True, False, False, "gauss"),
    (1, 2, 256, 128, False, False, False, "qknorm"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
    (2, 1, 256, 64, False, True, False, "qknorm"),
]


@pytest.mark.parametrize("B,H,N,d,causal,qs,u8,recipe", PCOL_CASES)
def test_fwd_bwd_parity_p_colscale(B, H, N, d, causal, qs, u8, recipe):
    """SAGE_P_COLSCALE (per-key psi(P) in the backward) against the oracle's ORC_P_COL mode, also
    combined with SAGE_P_U8."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=700 + N + d)
    gpu = _run(q, k, v, do, causal, True, qs, p_u8=u8, p_colscale=True)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, True, qs, p_u8=u8, p_col=True)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), ("pcol", B, H, N, d, causal, qs, u8, recipe))


FINE_CASES = [
    (1, 2, 384, 64, True, False, False, "gauss"),
    (1, 2, 256, 64, False, True, False, "outlier_kq"),
    (1, 2, 256, 128, False, False, False, "qknorm"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
    (2, 1, 512, 128, True, False, False, "gauss"),
]


@pytest.mark.parametrize("B,H,N,d,causal,qs,u8,recipe", FINE_CASES)
def test_fwd_bwd_parity_fine_bwd(B, H, N, d, causal, qs, u8, recipe):
    """SAGE_FINE_BWD (per-key psi(P), per-key dS^ for dK, per-query dS^ for dQ) against the oracle's
    ORC_P_COL | ORC_DS_FINE mode, also with Q-smoothing and SAGE_P_U8."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=800 + N + d)
    gpu = _run(q, k, v, do, causal, True, qs, p_u8=u8, fine_bwd=True)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, True, qs, p_u8=u8, p_col=True, ds_fine=True)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), ("fine", B, H, N, d, causal, qs, u8, recipe))


DET_CASES = [
    (1, 2, 512, 64, True, False),
    (1, 2, 384, 128, False, False),
    (1, 2, 384, 128, True, True),
]


@pytest.mark.parametrize("B,H,N,d,causal,qs", DET_CASES)
def test_deterministic_parity_and_repeatability(B, H, N, d, causal, qs):
    """SAGE_DETERMINISTIC (reading A19): three runs give bitwise identical O, dQ, dK, dV, and the
    result meets the same tolerance against the oracle."""
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq" if qs else "qknorm", seed=600 + N + d)
    runs = [_run(q, k, v, do, causal, True, qs, deterministic=True) for _ in range(3)]
    for r in runs[1:]:
        for name in ("o", "dq", "dk", "dv"):
            assert torch.equal(runs[0][name], r[name]), name
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, True, qs)
    _assert_ok(_compare(runs[0], f, b, heads, B, H, N, d), ("det", B, H, N, d, causal, qs))


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_deterministic_full_size_repeatable(cfg):
    """At the bench shapes (every CTA of a head racing for the same dQ rows) the deterministic dQ
    is bitwise identical across runs, and equal to the default path within the tolerance."""
    c = CONFIGS[cfg]
    q, k, v, do = make_inputs(c.batch, c.heads, c.seqlen, c.head_dim, c.recipe, seed=c.seed)
    r1 = _run(q, k, v, do, c.causal, c.k_smooth, c.q_smooth, deterministic=True)
    r2 = _run(q, k, v, do, c.causal, c.k_smooth, c.q_smooth, deterministic=True)
    assert torch.equal(r1["dq"], r2["dq"]) and torch.equal(r1["dk"], r2["dk"]) and torch.equal(r1["dv"], r2["dv"])
    r0 = _run(q, k, v, do, c.causal, c.k_smooth, c.q_smooth)
    assert rel_l2(f64(r0["dq"]), f64(r1["dq"])) < 1e-3


def test_zero_do_gives_zero_grads():
    """dO = 0: every dS tile is all-zero, scale 0 (reading A3) -> exact zeros."""
    q, k, v, do = make_inputs(1, 2, 256, 64, "gauss", seed=5)
    gpu = _run(q, k, v, torch.zeros_like(do), True, True, False)
    for name in ("dq", "dk", "dv"):
        assert torch.count_nonzero(gpu[name]).item() == 0


def test_autograd_function():
    q, k, v, do = (t.cuda() for t in make_inputs(1, 2, 256, 64, "qknorm", seed=6))
    q.requires_grad_(True)
    k.requires_grad_(True)
    v.requires_grad_(True)
    o = sage.sage_attention(q, k, v, causal=True)
    o.backward(do)
    o2, lse, ctx = sage.forward(q.detach(), k.detach(), v.detach(), causal=True)
    dq, dk, dv = sage.backward(ctx, v.detach(), o2, lse, do)
    assert torch.equal(o, o2)
    for g1, g2 in ((q.grad, dq), (k.grad, dk), (v.grad, dv)):
        assert rel_l2(f64(g2), f64(g1)) < 1e-3  # dQ reduction order differs run to run


# ------------------------------------------------------------------ full BASELINE sizes, sampled heads
@pytest.mark.parametrize("cfg,heads", [("C2", [0, 77, 127]), ("C3", [5, 126])])
def test_full_size_sampled_heads(cfg, heads):
    c = CONFIGS[cfg]
    q, k, v, do = make_inputs(c.batch, c.heads, c.seqlen, c.head_dim, c.recipe, seed=c.seed)
    gpu = _run(q, k, v, do, c.causal, c.k_smooth, c.q_smooth)
    oracle.set_threads(max(1, len(heads)))
    f, b = _oracle(q, k, v, do, heads, c.causal, c.k_smooth, c.q_smooth)
    _assert_ok(_compare(gpu, f, b, heads, c.batch, c.heads, c.seqlen, c.head_dim), cfg)


@pytest.mark.slow
@pytest.mark.parametrize("cfg,heads", [("C5", [3]), ("C4", [40])])
def test_full_size_long_sampled_head(cfg, heads):
    c = CONFIGS[cfg]
    q, k, v, do = make_inputs(c.batch, c.heads, c.seqlen, c.head_dim, c.recipe, seed=c.seed)
    gpu = _run(q, k, v, do, c.causal, c.k_smooth, c.q_smooth)
    f, b = _oracle(q, k, v, do, heads, c.causal, c.k_smooth, c.q_smooth)
    _assert_ok(_compare(gpu, f, b, heads, c.batch, c.heads, c.seqlen, c.head_dim), cfg)


# ------------------------------------------------------------------ QK-norm variant
QKN_CASES = [
    # (B, H, N, d, causal, k_smooth, q_smooth, fine_bwd)
    (1, 2, 384, 64, True, True, False, False),
    (1, 2, 256, 128, False, True, False, False),
    (1, 2, 384, 128, True, True, True, False),
    (1, 2, 256, 64, True, True, False, True),
]


def _qkn_inputs(B, H, N, d, seed):
    xq, xk, v, do = make_inputs(B, H, N, d, "noqknorm", seed=seed)
    g = torch.Generator().manual_seed(seed + 7)
    gq = (0.5 + 1.5 * torch.rand(d, generator=g)).float()
    gk = (0.5 + 1.5 * torch.rand(d, generator=g)).float()
    return xq, xk, v, do, gq, gk


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,fine", QKN_CASES)
def test_qknorm_parity(B, H, N, d, causal, ks, qs, fine):
    """sage_fwd_qknorm / sage_bwd_qknorm against oracle.qknorm + the quantised oracle:
    rstd, Q^, K^ and their scales bit-exact (Tier A: the fused normalisation produces exactly the
    bf16 Q, K of readings A24/A25); O, dX_q, dX_k, dV within the tolerance; dgamma likewise."""
    xq, xk, v, do, gq, gk = _qkn_inputs(B, H, N, d, seed=400 + N + d)
    dev = "cuda"
    xqd, xkd, vd, dod, gqd, gkd = (t.to(dev) for t in (xq, xk, v, do, gq, gk))
    o, lse, ctx = sage.forward_qknorm(xqd, xkd, vd, gqd, gkd, 1e-6, causal=causal, k_smooth=ks, q_smooth=qs,
                                      fine_bwd=fine)
    dxq, dxk, dv, dgq, dgk = sage.backward_qknorm(ctx, xqd, xkd, gqd, gkd, vd, o, lse, dod)
    torch.cuda.synchronize()
    BH = B * H
    flat = lambda t: f64(t).reshape(BH, N, d)
    qn_, rq = oracle.qknorm.forward(flat(xq), gq.numpy(), 1e-6)
    kn_, rk = oracle.qknorm.forward(flat(xk), gk.numpy(), 1e-6)
    view = ctx.view()
    np.testing.assert_array_equal(view["rstd_q"].cpu().numpy().reshape(BH, N), rq)
    np.testing.assert_array_equal(view["rstd_k"].cpu().numpy().reshape(BH, N), rk)
    kw = dict(causal=causal, k_smooth=ks, q_smooth=qs)
    f = oracle.fwd(qn_, kn_, flat(v), **kw)
    np.testing.assert_array_equal(view["q_i8"].cpu().numpy().reshape(BH, N, d), f["q8"])
    np.testing.assert_array_equal(view["k_i8"].cpu().numpy().reshape(BH, N, d), f["k8"])
    np.testing.assert_array_equal(view["q_scale"].cpu().numpy().reshape(BH, -1), f["sq"])
    np.testing.assert_array_equal(view["k_scale"].cpu().numpy().reshape(BH, -1), f["sk"])
    np.testing.assert_array_equal(view["mu_k"].cpu().numpy().reshape(BH, d), f["mu_k"])
    b = oracle.bwd(qn_, kn_, flat(v), round_bf16(f["o"]), flat(do), f["lse"], p_col=fine, ds_fine=fine, **kw)
    # A26: the module chain hands the bf16-rounded attention gradients to the RMSNorm backward
    dxq_r, dgq_r = oracle.qknorm.backward(flat(xq), gq.numpy(), rq, round_bf16(b["dq"]))
    dxk_r, dgk_r = oracle.qknorm.backward(flat(xk), gk.numpy(), rk, round_bf16(b["dk"]))
    for name, got, ref in (("o", o, f["o"]), ("dxq", dxq, dxq_r), ("dxk", dxk, dxk_r), ("dv", dv, b["dv"])):
        ref = round_bf16(ref)
        got = flat(got)
        rl, cs = rel_l2(ref, got), cos_sim(ref, got)
        assert rl <= REL_TOL and cs >= COS_TOL, (name, rl, cs)
    for name, got, ref in (("dgq", dgq, dgq_r), ("dgk", dgk, dgk_r)):
        got = f64(got)
        rl, cs = rel_l2(ref, got), cos_sim(ref, got)
        assert rl <= REL_TOL and cs >= COS_TOL, (name, rl, cs)


def test_qknorm_autograd_and_rejections():
    """The autograd wrapper returns the gamma gradients."""
    xq, xk, v, do, gq, gk = (t.cuda() for t in _qkn_inputs(1, 2, 256, 64, seed=9))
    for t in (xq, xk, v, gq, gk):
        t.requires_grad_(True)
    o = sage.sage_attention_qknorm(xq, xk, v, gq, gk, causal=True)
    o.backward(do)
    o2, lse, ctx = sage.forward_qknorm(xq.detach(), xk.detach(), v.detach(), gq.detach(), gk.detach(), causal=True)
    ref = sage.backward_qknorm(ctx, xq.detach(), xk.detach(), gq.detach(), gk.detach(), v.detach(), o2, lse, do)
    assert torch.equal(o, o2)
    for g1, g2 in zip((xq.grad, xk.grad, v.grad, gq.grad, gk.grad), ref):
        assert rel_l2(f64(g2), f64(g1)) < 1e-3



# ------------------------------------------------------------------ fp16 I/O (SAGE_FP16)
FP16_CASES = [
    (1, 2, 384, 64, True, True, False, "qknorm"),
    (1, 2, 256, 128, False, True, False, "gauss"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", FP16_CASES)
def test_fp16_parity(B, H, N, d, causal, ks, qs, recipe):
    """fp16 Q, K, V, dO (the paper's "FP16" dP option): Q^, K^ and their scales bit-exact
    (Tier A); O, dQ, dK, dV within the tolerance against the oracle, O stored as fp16 (A15) and both
    sides rounded to fp16 for the comparison (A18)."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=900 + N + d, dtype=torch.float16)
    gpu = _run(q, k, v, do, causal, ks, qs)
    assert gpu["o"].dtype == torch.float16 and gpu["dq"].dtype == torch.float16
    BH = B * H
    flat = lambda t: f64(t).reshape(BH, N, d)
    kw = dict(causal=causal, k_smooth=ks, q_smooth=qs)
    f = oracle.fwd(flat(q), flat(k), flat(v), **kw)
    b = oracle.bwd(flat(q), flat(k), flat(v), round_fp16(f["o"]), flat(do), f["lse"], **kw)
    view = gpu["ctx"].view()
    np.testing.assert_array_equal(view["q_i8"].cpu().numpy().reshape(BH, N, d), f["q8"])
    np.testing.assert_array_equal(view["k_i8"].cpu().numpy().reshape(BH, N, d), f["k8"])
    np.testing.assert_array_equal(view["k_scale"].cpu().numpy().reshape(BH, -1), f["sk"])
    for name, ref in (("o", f["o"]), ("dq", b["dq"]), ("dk", b["dk"]), ("dv", b["dv"])):
        ref = round_fp16(ref)
        got = flat(gpu[name])
        rl, cs = rel_l2(ref, got), cos_sim(ref, got)
        assert rl <= REL_TOL and cs >= COS_TOL, (name, rl, cs)


def test_fp16_qknorm_and_dtype_checks():
    """fp16 through the fused QK-norm (the module output is then fp16, A25) against the oracle, and
    the binding's dtype checks."""
    B, H, N, d = 1, 2, 256, 64
    xq, xk, v, do, gq, gk = _qkn_inputs(B, H, N, d, seed=77)
    xq, xk, v, do = (t.to(torch.float16) for t in (xq, xk, v, do))
    dev = "cuda"
    xqd, xkd, vd, dod, gqd, gkd = (t.to(dev) for t in (xq, xk, v, do, gq, gk))
    o, lse, ctx = sage.forward_qknorm(xqd, xkd, vd, gqd, gkd, 1e-6, causal=True)
    dxq, dxk, dv, dgq, dgk = sage.backward_qknorm(ctx, xqd, xkd, gqd, gkd, vd, o, lse, dod)
    torch.cuda.synchronize()
    flat = lambda t: f64(t).reshape(B * H, N, d)
    # the oracle's QK-norm with an fp16 module output (A25 with the I/O type)
    rq = oracle.qknorm.rstd(flat(xq), 1e-6)
    rk = oracle.qknorm.rstd(flat(xk), 1e-6)
    qn = round_fp16((flat(xq).astype(np.float32) * rq[..., None]).astype(np.float32) * gq.numpy())
    kn = round_fp16((flat(xk).astype(np.float32) * rk[..., None]).astype(np.float32) * gk.numpy())
    np.testing.assert_array_equal(ctx.view()["rstd_q"].cpu().numpy().reshape(B * H, N), rq)
    f = oracle.fwd(qn, kn, flat(v), causal=True)
    np.testing.assert_array_equal(ctx.view()["q_i8"].cpu().numpy().reshape(B * H, N, d), f["q8"])
    b = oracle.bwd(qn, kn, flat(v), round_fp16(f["o"]), flat(do), f["lse"], causal=True)
    dxq_r, _ = oracle.qknorm.backward(flat(xq), gq.numpy(), rq, round_fp16(b["dq"]))
    for name, got, ref in (("o", o, f["o"]), ("dxq", dxq, dxq_r), ("dv", dv, b["dv"])):
        rl = rel_l2(round_fp16(ref), flat(got))
        assert rl <= REL_TOL, (name, rl)
    with pytest.raises(sage.SageError):
        sage.forward(xqd, xkd.to(torch.bfloat16), vd)


def test_max_seqlen_properties():
    """N = 32768 (the metric's upper end, the library's kMaxSeqLen), properties that hold at any size:
    V = 1 gives O = 1 up to P^'s rounding (each row's P~ sums to l, P^ s_P to l within 1/254 per
    element); dO = 0 gives exactly zero gradients (all-zero dS tiles, reading A3); L is finite."""
    B, H, N, d = 1, 1, 32768, 128
    q, k, _, _ = make_inputs(B, H, N, d, "qknorm", seed=31)
    v = torch.ones_like(q)
    do = torch.zeros_like(q)
    gpu = _run(q, k, v, do, True, True, False)
    o = gpu["o"].float()
    assert torch.isfinite(gpu["lse"]).all()
    assert (o - 1.0).abs().max().item() < 0.02
    for name in ("dq", "dk", "dv"):
        assert torch.count_nonzero(gpu[name]).item() == 0, name


# ------------------------------------------------------------------ softmax scale, fp32 outputs, binding checks
@pytest.mark.parametrize("d,tau", [(64, 0.05), (128, 0.2)])
def test_non_default_softmax_scale(d, tau):
    """sage_params.softmax_scale (reading A6): S, dQ and dK carry the caller's tau."""
    B, H, N = 1, 2, 384
    q, k, v, do = make_inputs(B, H, N, d, "gauss", seed=70 + d, sigma=2.0)
    gpu = _run(q, k, v, do, True, True, False, softmax_scale=tau)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, True, True, False, tau=tau)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), ("tau", d, tau))
    # and it differs from the default scale's result
    g0 = _run(q, k, v, do, True, True, False)
    assert rel_l2(f64(g0["o"]), f64(gpu["o"])) > 1e-2


FP32_CASES = [
    (1, 2, 384, 64, True, True, False, "qknorm"),
    (1, 2, 256, 128, False, True, True, "outlier_kq"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", FP32_CASES)
def test_fp32_out_against_unrounded_oracle(B, H, N, d, causal, ks, qs, recipe):
    """SAGE_FP32_OUT (reading A18): O, dQ, dK, dV in fp32, compared against the oracle's unrounded double
    results (O stored as fp32 for delta, A15) -- without the bf16 rounding that takes 1.66e-3 of the budget
    the GPU is within 5e-4 of the quantised oracle."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=1300 + N + d)
    gpu = _run(q, k, v, do, causal, ks, qs, fp32_out=True)
    for n in ("o", "dq", "dk", "dv"):
        assert gpu[n].dtype == torch.float32, n
    heads = list(range(B * H))
    f32 = lambda x: np.asarray(x, np.float64).astype(np.float32).astype(np.float64)
    f, b = _oracle(q, k, v, do, heads, causal, ks, qs, o_round=f32)
    res = _compare(gpu, f, b, heads, B, H, N, d, out_round=lambda x: x)
    for name in ("o", "dq", "dk", "dv"):
        assert res[name][0] <= 5e-4 and res[name][1] >= 0.99999, (name, res)
    assert res["lse"] <= 1e-5, res


def test_binding_rejects_mismatched_tensors():
    """The binding checks shapes, dtypes and devices against the forward's context before calling the C
    ABI, and the C ABI refuses a context produced under other params (sage_ctx.params_tag)."""
    q, k, v, do = (t.cuda() for t in make_inputs(1, 2, 256, 64, "gauss", seed=3))
    o, lse, ctx = sage.forward(q, k, v, causal=True)
    with pytest.raises(sage.SageError):
        sage.backward(ctx, v[:, :1].contiguous(), o, lse, do[:, :1].contiguous())
    with pytest.raises(sage.SageError):
        sage.backward(ctx, v, o, lse[:, :1].contiguous(), do)
    with pytest.raises(sage.SageError):
        sage.forward(q, k, v, out=torch.empty(1, 2, 256, 64, dtype=torch.float32, device="cuda"))
    # a ctx from a non-causal forward presented with causal params: refused by the library
    o2, lse2, ctx2 = sage.forward(q, k, v, causal=False)
    ctx2.params = ctx.params
    with pytest.raises(sage.SageError, match="INVALID_VALUE"):
        sage.backward(ctx2, v, o2, lse2, do)
    # a context never filled by sage_fwd (tag 0)
    ctx3 = sage.SageCtx(ctx.params, torch.empty_like(ctx.buf), ctx.shape)
    with pytest.raises(sage.SageError, match="INVALID_VALUE"):
        sage.backward(ctx3, v, o, lse, do)


def test_streams_and_devices():
    """Calls on a side stream use that stream's own workspace and agree with the default stream's."""
    q, k, v, do = (t.cuda() for t in make_inputs(1, 2, 256, 128, "qknorm", seed=4))
    o, lse, ctx = sage.forward(q, k, v, causal=True)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        o2, lse2, ctx2 = sage.forward(q, k, v, causal=True)
        dq2, dk2, dv2 = sage.backward(ctx2, v, o2, lse2, do)
    torch.cuda.current_stream().wait_stream(s)
    dq, dk, dv = sage.backward(ctx, v, o, lse, do)
    torch.cuda.synchronize()
    assert torch.equal(o, o2) and torch.equal(lse, lse2) and torch.equal(dv, dv2) and torch.equal(dk, dk2)
    assert rel_l2(f64(dq), f64(dq2)) < 1e-3  # dQ's fp32 reduction order varies run to run
    keys = [key for key in sage._ws.bufs if key[1] == s.cuda_stream]
    assert keys, "the side stream got its own workspace"


@pytest.mark.slow
def test_max_seqlen_sampled_oracle_head():
    """N = 32768 (kMaxSeqLen, the top of the metric's 1K-32K) against the oracle on sampled blocks of one
    head: query blocks {0, 100, 255} (O, L, dQ) and key blocks {200, 255} (dK, dV); the oracle runs the
    same tiles as a full run for those rows (oracle.fwd / bwd q_blocks / k_blocks, pinned bitwise)."""
    B, H, N, d = 1, 1, 32768, 128
    q, k, v, do = make_inputs(B, H, N, d, "qknorm", seed=32)
    gpu = _run(q, k, v, do, True, True, False)
    qb, kb = [0, 100, 255], [200, 255]
    need = sorted(set(qb) | set(range(200, 256)))
    flat = lambda t: f64(t).reshape(1, N, d)
    oracle.set_threads(8)
    f = oracle.fwd(flat(q), flat(k), flat(v), causal=True, q_blocks=need)
    b = oracle.bwd(flat(q), flat(k), flat(v), round_bf16(f["o"]), flat(do), f["lse"], causal=True,
                   q_blocks=qb, k_blocks=kb)
    rows = lambda bl: np.concatenate([np.arange(i * 128, (i + 1) * 128) for i in bl])
    for name, ref, r in (("o", f["o"], rows(qb)), ("dq", b["dq"], rows(qb)), ("dk", b["dk"], rows(kb)),
                         ("dv", b["dv"], rows(kb))):
        got = flat(gpu[name])[0][r]
        want = round_bf16(ref[0][r])
        assert rel_l2(want, got) <= REL_TOL and cos_sim(want, got) >= COS_TOL, (name, rel_l2(want, got))
    lse = f64(gpu["lse"]).reshape(N)[rows(qb)]
    assert np.abs(lse - f["lse"][0][rows(qb)]).max() <= 1e-5


@pytest.mark.parametrize("d,causal,qs", [(64, False, False), (128, True, False), (128, False, True), (64, True, True)])
def test_repeatable_under_reuse(d, causal, qs):
    """Race evidence without a sanitizer (compute-sanitizer is closed on this pool): 12 back-to-back fwd+bwd
    runs on the same buffers must give bitwise identical O, L, dK, dV (every one of them is computed in a
    fixed order by one CTA; a missing barrier or a premature reuse of a pipeline buffer shows up as run-to-run
    differences), and dQ (an fp32 reduction in arrival order) within 1e-4 rel-L2 of the first run."""
    B, H, N = 2, 2, 640
    q, k, v, do = (t.cuda() for t in make_inputs(B, H, N, d, "outlier_kq", seed=90 + d))
    o, lse, ctx = sage.forward(q, k, v, causal=causal, q_smooth=qs)
    dq, dk, dv = sage.backward(ctx, v, o, lse, do)
    ref = [t.clone() for t in (o, lse, dq, dk, dv)]
    for _ in range(12):
        sage.forward(q, k, v, causal=causal, q_smooth=qs, out=o, lse=lse, ctx=ctx.buf)
        sage.backward(ctx, v, o, lse, do, dq=dq, dk=dk, dv=dv)
        torch.cuda.synchronize()
        for name, a, b in zip(("o", "lse", "dk", "dv"), ref[:2] + ref[3:], (o, lse, dk, dv)):
            assert torch.equal(a, b), name
        assert rel_l2(f64(ref[2]), f64(dq)) < 1e-4


# ------------------------------------------------------------------ FP8 E4M3 P^V^ (SAGE_PV_FP8, NEXT-4)
PV_FP8_CASES = [
    (1, 2, 384, 64, True, True, False, "qknorm"),
    (1, 2, 256, 128, False, True, False, "gauss"),
    (1, 2, 384, 128, True, True, True, "outlier_kq"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", PV_FP8_CASES)
def test_pv_fp8_parity(B, H, N, d, causal, ks, qs, recipe):
    """SAGE_PV_FP8 (reading A30) against the oracle's ORC_PV_FP8 mode: V^ in E4M3 and its scales bit-exact
    (Tier A, psi_block_e4m3 per 128-row block), O, L and the (unchanged) backward within the tolerance."""
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=1400 + N + d)
    dev = "cuda"
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, k_smooth=ks, q_smooth=qs, pv_fp8=True)
    dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
    torch.cuda.synchronize()
    BH, T = B * H, N // 128
    p = ctx.params
    wsf = sage._ws.get(p, False, torch.device(dev))
    wv = sage.ws_view(p, False, wsf)
    base = wsf.data_ptr()
    v8 = wsf[wv.v_i8 - base: wv.v_i8 - base + BH * N * d].view(torch.float8_e4m3fn).float().cpu().numpy()
    sv = wsf[wv.v_scale - base: wv.v_scale - base + BH * T * 4].view(torch.float32).cpu().numpy().reshape(BH, T)
    vf = f64(v).reshape(BH, N, d)
    for h in range(BH):
        for t in range(T):
            ref_q, ref_s = oracle.psi_block_e4m3(vf[h, t * 128:(t + 1) * 128])
            np.testing.assert_array_equal(v8.reshape(BH, N, d)[h, t * 128:(t + 1) * 128], ref_q)
            assert sv[h, t] == np.float32(ref_s)
    heads = list(range(BH))
    sel = lambda t: f64(t).reshape(BH, N, d)
    kw = dict(causal=causal, k_smooth=ks, q_smooth=qs)
    f = oracle.fwd(sel(q), sel(k), sel(v), pv_fp8=True, **kw)
    b = oracle.bwd(sel(q), sel(k), sel(v), round_bf16(f["o"]), sel(do), f["lse"], **kw)
    gpu = dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), ("pv_fp8", B, H, N, d, causal, qs))


# ------------------------------------------------------------------ strided I/O layouts (sage_params strides)
@pytest.mark.parametrize("d,causal,qs", [(64, True, False), (128, False, True), (128, True, False)])
def test_strided_bshd_layout(d, causal, qs):
    """Q, K, V, dO given as [B, N, H, d] tensors viewed as [B, H, N, d] (no copy: the library addresses rows
    through sage_params strides, 4-D TMA maps for V and dO): O, L, dK, dV bitwise identical to the contiguous
    run, dQ within its fp32 reduction-order noise, and the outputs come back in the inputs' layout."""
    B, H, N = 2, 2, 384
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=1600 + d)
    dev = "cuda"
    cont = [t.to(dev) for t in (q, k, v, do)]
    strided = [t.transpose(1, 2).contiguous().to(dev).transpose(1, 2) for t in (q, k, v, do)]
    assert not strided[0].is_contiguous()
    res = []
    for qd, kd, vd, dod in (cont, strided):
        o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, q_smooth=qs)
        dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
        torch.cuda.synchronize()
        res.append((o, lse, dq, dk, dv, ctx))
    (o0, l0, dq0, dk0, dv0, c0), (o1, l1, dq1, dk1, dv1, c1) = res
    assert c1.params.stride_n == H * d and o1.stride() == strided[0].stride() and dq1.stride() == strided[0].stride()
    assert torch.equal(o0, o1) and torch.equal(l0, l1) and torch.equal(dk0, dk1) and torch.equal(dv0, dv1)
    assert rel_l2(f64(dq0), f64(dq1)) < 1e-4


def test_strided_qknorm_and_fp32_out():
    """The strided layout through the fused QK-norm entry points and with SAGE_FP32_OUT (dQ then goes through
    the workspace accumulator and K5 into the strided fp32 output)."""
    B, H, N, d = 1, 2, 256, 128
    xq, xk, v, do, gq, gk = _qkn_inputs(B, H, N, d, seed=1700)
    dev = "cuda"
    gqd, gkd = gq.to(dev), gk.to(dev)
    outs = []
    for tr in (False, True):
        ts = [t.to(dev) if not tr else t.transpose(1, 2).contiguous().to(dev).transpose(1, 2) for t in (xq, xk, v, do)]
        o, lse, ctx = sage.forward_qknorm(ts[0], ts[1], ts[2], gqd, gkd, 1e-6, causal=True)
        g = sage.backward_qknorm(ctx, ts[0], ts[1], gqd, gkd, ts[2], o, lse, ts[3])
        of, lf, cf = sage.forward(ts[0], ts[1], ts[2], causal=True, fp32_out=True)
        gf = sage.backward(cf, ts[2], of, lf, ts[3])
        torch.cuda.synchronize()
        outs.append((o, lse) + tuple(g) + (of, lf) + tuple(gf))
    for a, b in zip(outs[0], outs[1]):  # dQ / dX_q and dgamma see the fp32 reduction order: tolerance
        assert rel_l2(f64(a), f64(b)) < 1e-4, (a.shape, rel_l2(f64(a), f64(b)))
