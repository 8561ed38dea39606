"""GPU parity at a sequence length that is not a multiple of the 128-row block (reading A33): the last block
of every head is short, its statistics are over the rows it holds, and the missing rows / columns of the
last tiles carry no logits.  Same contract as tests/test_gpu.py: Tier A bit-exact, outputs within the
north-star tolerance of the oracle (which implements A33 independently, pinned in tests/test_oracle.py)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_02170_b200 import sage
from paper_2603_02170_b200.inputs import make_inputs
from tests.metrics import cos_sim, f64, rel_l2, round_bf16
from tests.test_gpu import COS_TOL, REL_TOL, _assert_ok, _compare, _oracle, _qkn_inputs, _run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available() and torch.cuda.get_device_capability() == (10, 0)
    sage.lib()
    oracle.build()


def _ws_slice(buf, addr, n, dtype):
    base = buf.data_ptr()
    nbytes = n * torch.empty((), dtype=dtype).element_size()
    return buf[addr - base: addr - base + nbytes].view(dtype)


@pytest.mark.parametrize("N,d,q_smooth", [(300, 64, False), (300, 128, True), (129, 128, False)])
def test_ragged_tier_a(N, d, q_smooth):
    """Q^, K^, V^, dO^ and their scales, mu_K, mu_Q bit-exact, the bias within 1e-5, delta bit-exact; the padded
    rows of the library's buffers (Np = 128 ceil(N / 128) per head) are zero."""
    B, H = 1, 2
    BH, T = B * H, -(-N // 128)
    Np = T * 128
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=2100 + N + d)
    gpu = _run(q, k, v, do, True, True, q_smooth)
    view = gpu["ctx"].view()
    f, b = _oracle(q, k, v, do, list(range(BH)), True, True, q_smooth)
    q8 = view["q_i8"].cpu().numpy().reshape(BH, Np, d)
    k8 = view["k_i8"].cpu().numpy().reshape(BH, Np, d)
    np.testing.assert_array_equal(q8[:, :N], f["q8"])
    np.testing.assert_array_equal(k8[:, :N], f["k8"])
    assert not q8[:, N:].any() and not k8[:, N:].any()
    np.testing.assert_array_equal(view["q_scale"].cpu().numpy().reshape(BH, T), f["sq"])
    np.testing.assert_array_equal(view["k_scale"].cpu().numpy().reshape(BH, T), f["sk"])
    np.testing.assert_array_equal(view["mu_k"].cpu().numpy().reshape(BH, d), f["mu_k"])
    if q_smooth:
        np.testing.assert_array_equal(view["mu_q"].cpu().numpy().reshape(BH, T, d), f["mu_q"])
        bias = view["bias"].cpu().numpy().reshape(BH, T, Np).astype(np.float64)
        assert np.abs(bias[:, :, :N] - f["bias"]).max() <= 1e-5 * np.abs(f["bias"]).max()
        assert not bias[:, :, N:].any()
    p = gpu["ctx"].params
    wsf = sage._ws.get(p, False, torch.device("cuda"))
    wv = sage.ws_view(p, False, wsf)
    v8 = _ws_slice(wsf, wv.v_i8, BH * Np * d, torch.int8).cpu().numpy().reshape(BH, Np, d)
    np.testing.assert_array_equal(v8[:, :N], f["v8"])
    assert not v8[:, N:].any()
    np.testing.assert_array_equal(_ws_slice(wsf, wv.v_scale, BH * T, torch.float32).cpu().numpy().reshape(BH, T),
                                  f["sv"])
    wsb = sage._ws.get(p, True, torch.device("cuda"))
    wb = sage.ws_view(p, True, wsb)
    do8 = _ws_slice(wsb, wb.do_i8, BH * Np * d, torch.int8).cpu().numpy().reshape(BH, Np, d)
    np.testing.assert_array_equal(do8[:, :N], b["do8"])
    np.testing.assert_array_equal(_ws_slice(wsb, wb.do_scale, BH * T, torch.float32).cpu().numpy().reshape(BH, T),
                                  b["sdo"])
    delta = _ws_slice(wsb, wb.delta, BH * Np, torch.float32).cpu().numpy().reshape(BH, Np)
    flat = lambda t: f64(t).reshape(BH, N, d)
    b_st = oracle.bwd(flat(q), flat(k), flat(v), flat(gpu["o"]), flat(do), f["lse"], causal=True, k_smooth=True,
                      q_smooth=q_smooth)
    np.testing.assert_array_equal(delta[:, :N], b_st["delta"].astype(np.float32))
    assert not delta[:, N:].any()


RAGGED = [
    # (B, H, N, d, causal, k_smooth, q_smooth, recipe)
    (1, 2, 200, 64, True, True, False, "outlier_k"),
    (1, 2, 129, 64, False, True, False, "gauss"),
    (1, 2, 300, 128, True, True, True, "outlier_kq"),
    (1, 2, 1000, 128, False, True, False, "qknorm"),
    (2, 1, 257, 128, False, True, True, "outlier_kq"),
    (1, 2, 703, 64, True, True, True, "outlier_kq"),
    (1, 2, 100, 128, True, False, False, "gauss"),
]


@pytest.mark.parametrize("B,H,N,d,causal,ks,qs,recipe", RAGGED)
def test_ragged_parity(B, H, N, d, causal, ks, qs, recipe):
    q, k, v, do = make_inputs(B, H, N, d, recipe, seed=2200 + N + d)
    gpu = _run(q, k, v, do, causal, ks, qs)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, ks, qs)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), (B, H, N, d, causal, ks, qs, recipe))


@pytest.mark.parametrize("variant", ["p_u8", "fp32_out", "deterministic", "fine_bwd", "p_colscale", "pv_fp8"])
def test_ragged_variants(variant):
    """Each flag variant at a ragged N (N = 300, d = 128, causal, Q-smoothing) against its oracle mode."""
    B, H, N, d = 1, 2, 300, 128
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=2300)
    dev = "cuda"
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    kw = {variant: True}
    o, lse, ctx = sage.forward(qd, kd, vd, causal=True, q_smooth=True, **kw)
    dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
    torch.cuda.synchronize()
    heads = list(range(B * H))
    sel = lambda t: f64(t).reshape(B * H, N, d)
    okw = dict(causal=True, k_smooth=True, q_smooth=True)
    fo = oracle.fwd(sel(q), sel(k), sel(v), p_u8=variant == "p_u8", pv_fp8=variant == "pv_fp8", **okw)
    rnd = (lambda x: x) if variant == "fp32_out" else round_bf16
    bo = oracle.bwd(sel(q), sel(k), sel(v), rnd(fo["o"]), sel(do), fo["lse"], p_u8=variant == "p_u8",
                    p_col=variant in ("p_colscale", "fine_bwd"), ds_fine=variant == "fine_bwd", **okw)
    gpu = dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    _assert_ok(_compare(gpu, fo, bo, heads, B, H, N, d, out_round=rnd), variant)


def test_ragged_qknorm_and_strided():
    """The fused QK-norm entry points and a [B, N, H, d] strided layout at a ragged N."""
    B, H, N, d = 1, 2, 200, 128
    xq, xk, v, do, gq, gk = _qkn_inputs(B, H, N, d, seed=2400)
    dev = "cuda"
    xqd, xkd, vd, dod, gqd, gkd = (t.to(dev) for t in (xq, xk, v, do, gq, gk))
    o, lse, ctx = sage.forward_qknorm(xqd, xkd, vd, gqd, gkd, 1e-6, causal=True)
    dxq, dxk, dv, dgq, dgk = sage.backward_qknorm(ctx, xqd, xkd, gqd, gkd, vd, o, lse, dod)
    torch.cuda.synchronize()
    BH = B * H
    flat = lambda t: f64(t).reshape(BH, N, d)
    qn_, rq = oracle.qknorm.forward(flat(xq), gq.numpy(), 1e-6)
    kn_, rk = oracle.qknorm.forward(flat(xk), gk.numpy(), 1e-6)
    Np = -(-N // 128) * 128
    view = ctx.view()
    np.testing.assert_array_equal(view["rstd_q"].cpu().numpy().reshape(BH, Np)[:, :N], rq)
    np.testing.assert_array_equal(view["rstd_k"].cpu().numpy().reshape(BH, Np)[:, :N], rk)
    kw = dict(causal=True, k_smooth=True, q_smooth=False)
    f = oracle.fwd(qn_, kn_, flat(v), **kw)
    np.testing.assert_array_equal(view["q_i8"].cpu().numpy().reshape(BH, Np, d)[:, :N], f["q8"])
    b = oracle.bwd(qn_, kn_, flat(v), round_bf16(f["o"]), flat(do), f["lse"], **kw)
    dxq_r, dgq_r = oracle.qknorm.backward(flat(xq), gq.numpy(), rq, round_bf16(b["dq"]))
    dxk_r, dgk_r = oracle.qknorm.backward(flat(xk), gk.numpy(), rk, round_bf16(b["dk"]))
    for name, got, ref in (("o", o, f["o"]), ("dxq", dxq, dxq_r), ("dxk", dxk, dxk_r), ("dv", dv, b["dv"]),
                           ("dgq", dgq, dgq_r), ("dgk", dgk, dgk_r)):
        ref = round_bf16(ref) if name not in ("dgq", "dgk") else ref
        got = flat(got) if name not in ("dgq", "dgk") else f64(got)
        rl, cs = rel_l2(ref, got), cos_sim(ref, got)
        assert rl <= REL_TOL and cs >= COS_TOL, (name, rl, cs)
    # the same attention in a [B, N, H, d] layout: bitwise the contiguous result except dQ (reduction order)
    q, k, v2, do2 = make_inputs(B, H, N, d, "outlier_kq", seed=2401)
    res = []
    for tr in (False, True):
        ts = [t.to(dev) if not tr else t.transpose(1, 2).contiguous().to(dev).transpose(1, 2) for t in (q, k, v2, do2)]
        o2, l2, c2 = sage.forward(ts[0], ts[1], ts[2], causal=True, q_smooth=True)
        res.append((o2, l2) + tuple(sage.backward(c2, ts[2], o2, l2, ts[3])))
    torch.cuda.synchronize()
    for i, (a, b_) in enumerate(zip(res[0], res[1])):
        if i == 2:
            assert rel_l2(f64(a), f64(b_)) < 1e-4
        else:
            assert torch.equal(a, b_), i


def test_ragged_degenerate_lengths():
    """N = 1 (one key: P = 1, O = V^ dequantised, dS = dP - delta) and N = 127 (one short block) against
    the oracle; every output finite."""
    for N, d in ((1, 64), (127, 128)):
        q, k, v, do = make_inputs(1, 2, N, d, "gauss", seed=2500 + N)
        gpu = _run(q, k, v, do, True, True, False)
        f, b = _oracle(q, k, v, do, [0, 1], True, True, False)
        for name, ref in (("o", f["o"]), ("dq", b["dq"]), ("dk", b["dk"]), ("dv", b["dv"])):
            got = f64(gpu[name]).reshape(2, N, d)
            assert np.isfinite(got).all(), (N, name)
            scale = max(np.abs(round_bf16(ref)).max(), 1e-3)
            assert np.abs(got - round_bf16(ref)).max() <= 2e-2 * scale, (N, name)
        assert np.abs(f64(gpu["lse"]).reshape(2, N) - f["lse"]).max() <= 1e-5


@pytest.mark.parametrize("shape", [(0, 2, 256, 64), (1, 0, 256, 128), (1, 2, 0, 64)])
def test_empty_inputs(shape):
    """An empty batch, head count or sequence: empty results of the right shapes, forward and backward, and the
    autograd path; nothing is launched (the C ABI rejects empty shapes, so the binding returns early)."""
    q, k, v, do = (torch.zeros(shape, dtype=torch.bfloat16, device="cuda") for _ in range(4))
    o, lse, ctx = sage.forward(q, k, v, causal=True)
    assert o.shape == shape and lse.shape == shape[:3]
    dq, dk, dv = sage.backward(ctx, v, o, lse, do)
    assert dq.shape == dk.shape == dv.shape == shape
    qa = q.clone().requires_grad_()
    out = sage.sage_attention(qa, k, v, causal=True)
    out.sum().backward()
    assert out.shape == shape and qa.grad.shape == shape
    g = torch.ones(shape[3], dtype=torch.float32, device="cuda")
    o, lse, ctx = sage.forward_qknorm(q, k, v, g, g, 1e-6, causal=True)
    dxq, dxk, dv, dgq, dgk = sage.backward_qknorm(ctx, q, k, g, g, v, o, lse, do)
    assert dxq.shape == shape and dgq.shape == (shape[3],) and not dgq.any()


def test_ragged_max_length_sampled():
    """N = 32767 (the largest ragged length: 256 blocks, the last one 127 rows) against the oracle on sampled
    blocks of one head, with Q-smoothing: query blocks {0, 131, 255} (O, L, dQ; 255 is the short block) and
    key blocks {254, 255} (dK, dV); the oracle's sampled mode runs the same tiles as a full run."""
    B, H, N, d = 1, 1, 32767, 128
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=2600)
    gpu = _run(q, k, v, do, True, True, True)
    qb, kb = [0, 131, 255], [254, 255]
    need = sorted(set(qb) | set(range(254, 256)))
    flat = lambda t: f64(t).reshape(1, N, d)
    oracle.set_threads(8)
    kw = dict(causal=True, k_smooth=True, q_smooth=True)
    f = oracle.fwd(flat(q), flat(k), flat(v), q_blocks=need, **kw)
    b = oracle.bwd(flat(q), flat(k), flat(v), round_bf16(f["o"]), flat(do), f["lse"], q_blocks=qb, k_blocks=kb, **kw)
    rows = lambda bl: np.concatenate([np.arange(i * 128, min((i + 1) * 128, N)) for i in bl])
    for name, ref, r in (("o", f["o"], rows(qb)), ("dq", b["dq"], rows(qb)), ("dk", b["dk"], rows(kb)),
                         ("dv", b["dv"], rows(kb))):
        got = flat(gpu[name])[0][r]
        want = round_bf16(ref[0][r])
        assert rel_l2(want, got) <= REL_TOL and cos_sim(want, got) >= COS_TOL, (name, rel_l2(want, got))
    lse = f64(gpu["lse"]).reshape(N)[rows(qb)]
    assert np.abs(lse - f["lse"][0][rows(qb)]).max() <= 1e-5


def test_ragged_deterministic_noncausal():
    """SAGE_DETERMINISTIC's rotated non-causal order (CTA j visits query blocks (j + it) mod T, T = ceil(N/128)) at
    a ragged N: within the tolerance of the oracle, and dQ bitwise identical across two runs."""
    B, H, N, d = 1, 2, 300, 64
    q, k, v, do = make_inputs(B, H, N, d, "qknorm", seed=2700)
    runs = [_run(q, k, v, do, False, True, False, deterministic=True) for _ in range(2)]
    assert torch.equal(runs[0]["dq"], runs[1]["dq"])
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, False, True, False)
    _assert_ok(_compare(runs[0], f, b, heads, B, H, N, d), "det ragged")
