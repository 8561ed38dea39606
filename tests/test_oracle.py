"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Each test names the passage it pins.  A plausible mistake in the oracle (a dropped
term, a wrong sign or index, a transposed operand) must fail at least one of these.
"""
import math
import os

import numpy as np
import pytest
import torch

from paper_2603_02170_b200.inputs import make_inputs
from tests.metrics import cos_sim, f64, rel_l2, rms

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(rng, *shape, scale=1.0):
    """fp32-exact random doubles (the oracle's quantised mode sees FP32 numbers)."""
    return (rng.standard_normal(shape) * scale).astype(np.float32).astype(np.float64)


def _golden_psi():
    rows = []
    for line in open(os.path.join(GOLDEN, "psi_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        kind, inp, scale, vals = [f.strip() for f in line.split("|")]
        parse = lambda s: np.array([[float(x) for x in r.split()] for r in s.split(";")])
        rows.append((kind, parse(inp), scale, parse(vals)))
    return rows


# --------------------------------------------------------------------------- psi
def test_psi_worked_examples(orc):
    """SPEC S:129-130 / P:110-114 worked examples, and the per-token example S:150."""
    for kind, x, scale, vals in _golden_psi():
        if kind == "block":
            q, s = orc.psi_block(x)
            assert s == float(scale)
            np.testing.assert_array_equal(q, vals.astype(np.int8))
        else:
            q, sp = orc.psi_token_row(x.ravel(), 0.0)
            assert sp == pytest.approx(1.0 / 127.0, rel=1e-15)
            np.testing.assert_array_equal(q, vals.ravel().astype(np.int8))


def test_psi_half_step_bound_and_saturation(orc):
    """|x - q*scale| <= scale/2 (+fp32 slack, A4) and max|q| = 127 for nonzero blocks."""
    rng = np.random.default_rng(0)
    for trial in range(200):
        x = _rand(rng, 128, 64, scale=10.0 ** rng.uniform(-6, 3))
        q, s = orc.psi_block(x)
        assert np.abs(q.astype(int)).max() == 127
        assert s == pytest.approx(np.abs(x).max() / 127.0, rel=2 ** -23)
        err = np.abs(x - q.astype(np.float64) * s)
        assert err.max() <= s * (0.5 + 2 ** -15)


def test_psi_grid_fixed_point(orc):
    """Quantise-dequantise of a block already on the grid {-127s..127s} is exact."""
    rng = np.random.default_rng(1)
    ints = rng.integers(-127, 128, size=(128, 64)).astype(np.float64)
    ints[0, 0] = 127
    q, s = orc.psi_block(ints * 0.5)          # power-of-two scale: exactly representable grid
    assert s == np.float32(127 * 0.5) / np.float32(127)
    np.testing.assert_array_equal(q.astype(np.float64), ints)


def test_psi_token_row_properties(orc):
    """Row owning the running max reaches 127; scale e^{rm-m}/127; S:151 case."""
    rng = np.random.default_rng(2)
    s = rng.standard_normal(128)
    m = s.max()
    q, sp = orc.psi_token_row(np.exp(s - m), 0.0)
    assert q.max() == 127 and q.min() >= 0
    # rm - m = -ln(127): scales 1/127^2, entries <= 1/127 stay <= 127, no clamping.
    pt = np.exp(s - s.max()) / 127.0
    q, sp = orc.psi_token_row(pt, -math.log(127.0))
    assert sp == pytest.approx(1.0 / 127.0 ** 2, rel=1e-12)
    assert q.max() == 127


# --------------------------------------------------------------------------- FPA
@pytest.mark.parametrize("causal", [False, True])
def test_fpa_finite_differences(orc, causal):
    """FPA gradients == central finite differences of L = sum(O o G), step 1e-5."""
    for N, d in [(4, 2), (8, 4)]:
        for seed in range(5):
            rng = np.random.default_rng(100 + seed)
            q, k, v, g = (rng.standard_normal((1, N, d)) for _ in range(4))
            out = orc.fpa(q, k, v, g, causal=causal)
            for name, x in (("dq", q), ("dk", k), ("dv", v)):
                fd = np.zeros_like(x)
                for idx in np.ndindex(x.shape):
                    xp, xm = x.copy(), x.copy()
                    xp[idx] += 1e-5
                    xm[idx] -= 1e-5
                    args = dict(q=q, k=k, v=v)
                    args[name[1]] = xp
                    lp = (orc.fpa(**args, causal=causal)["o"] * g).sum()
                    args[name[1]] = xm
                    lm = (orc.fpa(**args, causal=causal)["o"] * g).sum()
                    fd[idx] = (lp - lm) / 2e-5
                assert rel_l2(fd, out[name]) <= 1e-5, (name, N, d, seed)


def test_fpa_closed_forms(orc):
    """N=1 -> O = V; Q=K=V=0 -> uniform P, O = 0; rows of P sum to 1."""
    rng = np.random.default_rng(3)
    v = rng.standard_normal((1, 1, 8))
    out = orc.fpa(rng.standard_normal((1, 1, 8)), rng.standard_normal((1, 1, 8)), v)
    np.testing.assert_allclose(out["o"], v, rtol=0, atol=1e-15)
    z = np.zeros((1, 4, 2))
    out = orc.fpa(z, z, z, intermediates=True)
    np.testing.assert_allclose(out["P"], 0.25, atol=1e-15)
    np.testing.assert_allclose(out["o"], 0.0, atol=1e-15)
    np.testing.assert_allclose(out["lse"], math.log(4), atol=1e-15)
    out = orc.fpa(*(rng.standard_normal((2, 32, 8)) for _ in range(3)), causal=True, intermediates=True)
    np.testing.assert_allclose(out["P"].sum(-1), 1.0, atol=1e-12)
    assert np.all(np.triu(out["P"][0], 1) == 0.0)


def test_ds_bound_appendix_b(orc):
    """App. B: RMS(dS) <= max_i ||dP_i - delta_i||_inf / sqrt(N); RMS(P_i) <= 1/sqrt(N)
    (P:748-755); dS rows sum to 0.  dO = 0 gives lhs = rhs = 0."""
    rng = np.random.default_rng(4)
    for N in (16, 64, 256):
        for d in (8, 64):
            for sigma in (1.0, 5.0, 10.0):
                q, k = (sigma * rng.standard_normal((1, N, d)) for _ in range(2))
                v, do = (rng.standard_normal((1, N, d)) for _ in range(2))
                out = orc.fpa(q, k, v, do, intermediates=True)
                P, dP, dS, delta = out["P"][0], out["dP"][0], out["dS"][0], out["delta"][0]
                rhs = np.abs(dP - delta[:, None]).max() / math.sqrt(N)
                assert rms(dS) <= rhs + 1e-15
                assert np.all(np.sqrt((P * P).mean(-1)) <= 1 / math.sqrt(N) + 1e-12)
                assert np.abs(dS.sum(-1)).max() <= 1e-9 * np.abs(dS).max() + 1e-12
    z = np.zeros((1, 16, 8))
    out = orc.fpa(rng.standard_normal((1, 16, 8)), rng.standard_normal((1, 16, 8)), z, z, intermediates=True)
    assert rms(out["dS"]) == 0.0


# --------------------------------------------------------------------------- tiled, quantisation off
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("smooth", ["none", "k", "qk"])
@pytest.mark.parametrize("N,blk", [(64, 16), (64, 32), (96, 32), (128, 128), (80, 32), (50, 16), (33, 32)])
def test_tiled_quant_off_equals_fpa(orc, causal, smooth, N, blk):
    """Alg. 1/2 with psi = identity == naive attention <= 1e-9.
    With smoothing this also pins: K-smoothing invariance, the
    four-term decomposition with the bias added back and
    dK = dK_center + dK_bias."""
    rng = np.random.default_rng(5)
    d = 16
    q = rng.standard_normal((2, N, d)) + rng.standard_normal(d) * 3
    k = rng.standard_normal((2, N, d)) + rng.standard_normal(d) * 5
    v, do = rng.standard_normal((2, N, d)), rng.standard_normal((2, N, d))
    ref = orc.fpa(q, k, v, do, causal=causal)
    kw = dict(causal=causal, k_smooth=smooth != "none", q_smooth=smooth == "qk", quant=False, blk=blk)
    f = orc.fwd(q, k, v, **kw)
    assert rel_l2(ref["o"], f["o"]) <= 1e-9
    # smoothing drops the row-constant terms Q_sm mu_K^T + mu_Q mu_K^T = Q mu_K^T,
    # so L of the smoothed logits is L_FPA - tau * Q_r . mu_K
    shift = np.einsum("bnd,bd->bn", q, k.mean(1)) / math.sqrt(d) if smooth != "none" else 0.0
    np.testing.assert_allclose(f["lse"] + shift, ref["lse"], rtol=0, atol=1e-8)
    b = orc.bwd(q, k, v, f["o"], do, f["lse"], **kw)
    for name in ("dq", "dk", "dv"):
        assert rel_l2(ref[name], b[name]) <= 1e-9, name


# --------------------------------------------------------------------------- ragged N (reading A33)
@pytest.mark.parametrize("N,d,mode", [(200, 64, "int8"), (300, 128, "int8"), (129, 64, "int8"), (200, 64, "p_u8"),
                                      (300, 64, "pv_fp8"), (200, 64, "p_col"), (300, 64, "ds_fine")])
def test_ragged_causal_prefix(orc, N, d, mode):
    """A causal ragged-N run is the first N rows of the padded run: zero rows appended to Q, K, V and dO
    change no block's psi scale (amax over zeros), and causal rows never see the later keys, so O, L, dQ and
    dK of the first N rows are bit-identical; dV only through the P^ tile scales (padded queries).  The same
    holds in every variant mode (P_U8, PV_FP8, P_COL, DS_FINE: the padded queries' dS is 0)."""
    rng = np.random.default_rng(N)
    BH, Np = 2, -(-N // 128) * 128
    q, k, v, do = (_rand(rng, BH, N, d) for _ in range(4))
    pad = lambda x: np.concatenate([x, np.zeros((BH, Np - N, d))], 1)
    fkw = dict(causal=True, k_smooth=False, p_u8=mode == "p_u8", pv_fp8=mode == "pv_fp8")
    bkw = dict(causal=True, k_smooth=False, p_u8=mode == "p_u8", p_col=mode in ("p_col", "ds_fine"),
               ds_fine=mode == "ds_fine")
    f = orc.fwd(q, k, v, **fkw)
    fp = orc.fwd(pad(q), pad(k), pad(v), **fkw)
    np.testing.assert_array_equal(f["o"], fp["o"][:, :N])
    np.testing.assert_array_equal(f["lse"], fp["lse"][:, :N])
    np.testing.assert_array_equal(f["sq"], fp["sq"])
    b = orc.bwd(q, k, v, f["o"], do, f["lse"], **bkw)
    bp = orc.bwd(pad(q), pad(k), pad(v), fp["o"], pad(do), fp["lse"], **bkw)
    np.testing.assert_array_equal(b["dq"], bp["dq"][:, :N])
    np.testing.assert_array_equal(b["dk"], bp["dk"][:, :N])
    assert rel_l2(bp["dv"][:, :N], b["dv"]) < 2e-3


def test_ragged_block_statistics(orc):
    """The short last block's statistics are over the rows it holds (A33): mu_K over all N rows, mu_Qi over
    the block's rows, and s = fl32(amax / 127) over them."""
    rng = np.random.default_rng(3)
    N, d = 300, 64
    q, k, v = (_rand(rng, 1, N, d) + 2.0 for _ in range(3))
    out = orc.fwd(q, k, v, causal=False, k_smooth=True, q_smooth=True)
    mu_k = np.array([math.fsum(k[0, :, c]) / N for c in range(d)], dtype=np.float32)
    np.testing.assert_array_equal(out["mu_k"][0], mu_k)
    last = q[0, 256:]
    mu_q = np.array([math.fsum(last[:, c]) / 44 for c in range(d)], dtype=np.float32)
    np.testing.assert_array_equal(out["mu_q"][0, 2], mu_q)
    qsm = last.astype(np.float32) - mu_q
    assert out["sq"][0, 2] == np.float32(np.float32(np.abs(qsm).max()) / np.float32(127))
    ksm = k[0, 256:].astype(np.float32) - mu_k
    assert out["sk"][0, 2] == np.float32(np.float32(np.abs(ksm).max()) / np.float32(127))
    assert out["sv"][0, 2] == np.float32(np.float32(np.abs(v[0, 256:]).max()) / np.float32(127))
    assert np.abs(out["q8"][0, 256:]).max() == 127 and out["o"].shape == (1, N, d)


# --------------------------------------------------------------------------- tiled, quantised (the QO)
def test_quant_mu_and_blocks(orc):
    """mu_K = exact column mean over all N tokens, rounded once to fp32 (A12, A17);
    every 128 x d block of K_sm, V satisfies the psi contract."""
    q, k, v, do = make_inputs(1, 2, 512, 64, "outlier_k", seed=7)
    q, k, v = f64(q), f64(k), f64(v)
    out = orc.fwd(q.reshape(2, 512, 64), k.reshape(2, 512, 64), v.reshape(2, 512, 64), causal=True)
    for h in range(2):
        kh = k[0, h]
        mu = np.array([math.fsum(kh[:, c]) / 512 for c in range(64)], dtype=np.float32)
        np.testing.assert_array_equal(out["mu_k"][h], mu)
        ksm = (kh.astype(np.float32) - mu).astype(np.float64)
        for t in range(4):
            blkk = ksm[t * 128:(t + 1) * 128]
            q8 = out["k8"][h, t * 128:(t + 1) * 128].astype(np.float64)
            s = float(out["sk"][h, t])
            assert np.abs(q8).max() == 127
            assert np.abs(blkk - q8 * s).max() <= s * (0.5 + 2 ** -15)
            vb = v[0, h, t * 128:(t + 1) * 128]
            v8 = out["v8"][h, t * 128:(t + 1) * 128].astype(np.float64)
            assert np.abs(vb - v8 * float(out["sv"][h, t])).max() <= float(out["sv"][h, t]) * (0.5 + 2 ** -15)


def test_quant_lse_is_logsumexp_of_quantised_logits(orc):
    """L_i = m + log l (Alg. 1 line 14, A7) equals the direct logsumexp of the dequantised
    INT8 logits S = (Q^ K^T) s_Q s_K tau (line 7, A6), causal mask (A14)."""
    q, k, v, _ = (f64(t).reshape(1, 384, 64) for t in make_inputs(1, 1, 384, 64, "gauss", seed=8, sigma=3.0))
    out = orc.fwd(q, k, v, causal=True)
    q8, k8 = out["q8"][0].astype(np.int64), out["k8"][0].astype(np.int64)
    sq, sk = np.repeat(out["sq"][0].astype(np.float64), 128), np.repeat(out["sk"][0].astype(np.float64), 128)
    S = (q8 @ k8.T).astype(np.float64) * sq[:, None] * sk[None, :] / 8.0
    S[np.triu_indices(384, 1)] = -np.inf
    mx = S.max(1)
    lse = mx + np.log(np.exp(S - mx[:, None]).sum(1))
    np.testing.assert_allclose(out["lse"][0], lse, rtol=0, atol=1e-9)
    # O approximates softmax(S) V up to the P~ / V quantisation (half-step bounds)
    P = np.exp(S - lse[:, None])
    assert rel_l2(P @ v[0], out["o"][0]) < 0.02


def test_quant_zero_do_gives_zero_grads(orc):
    """dO = 0 -> dQ = dK = dV = 0 exactly (all-zero blocks, A3)."""
    q, k, v, _ = (f64(t).reshape(2, 256, 64) for t in make_inputs(1, 2, 256, 64, "gauss", seed=9))
    f = orc.fwd(q, k, v, causal=True)
    b = orc.bwd(q, k, v, f["o"], np.zeros_like(q), f["lse"], causal=True)
    for name in ("dq", "dk", "dv"):
        assert np.all(b[name] == 0.0)


def _fidelity(orc, q, k, v, do, **kw):
    ref = orc.fpa(q, k, v, do, causal=kw.get("causal", False))
    f = orc.fwd(q, k, v, **kw)
    o_st = f["o"]
    b = orc.bwd(q, k, v, o_st, do, f["lse"], **kw)
    res = {"o": (cos_sim(ref["o"], f["o"]), rel_l2(ref["o"], f["o"]))}
    for name in ("dq", "dk", "dv"):
        res[name] = (cos_sim(ref[name], b[name]), rel_l2(ref[name], b[name]))
    return res


def _table1():
    rows = {}
    for line in open(os.path.join(GOLDEN, "table1_qkstd.txt")):
        if line.startswith("#") or not line.strip():
            continue
        f = [float(x) for x in line.split()]
        rows[f[0]] = {"o": f[1:3], "dq": f[3:5], "dk": f[5:7], "dv": f[7:9]}
    return rows


@pytest.mark.slow
def test_table1_sigma_sweep(orc):
    """Table 1: SageBwd vs FPA on Gaussian Q, K with sigma in {1,3,5,8,10}.
    The paper does not state N or d; at N = 1024, d = 64 (non-causal, K-smoothing on,
    P:405) the oracle must (a) grow strictly in sigma for every tensor and
    (b) land within the bands below of the paper's values (band evidence: DESIGN.md 3.3)."""
    tab = _table1()
    res = {}
    for sigma in (1.0, 3.0, 5.0, 8.0, 10.0):
        q, k, v, do = (f64(t).reshape(1, 1024, 64) for t in
                       make_inputs(1, 1, 1024, 64, "gauss", seed=11, sigma=sigma))
        res[sigma] = _fidelity(orc, q, k, v, do)
    sig = sorted(res)
    for name in ("o", "dq", "dk", "dv"):
        # dV at sigma = 1 sits above sigma = 3 under the literal per-tile psi(P) (reading A11)
        start = 1 if name == "dv" else 0
        rels = [res[s][name][1] for s in sig[start:]]
        assert all(a < b for a, b in zip(rels, rels[1:])), (name, rels)
    for s in sig:
        for name in ("o", "dq", "dk", "dv"):
            paper = tab[s][name][1]
            got = res[s][name][1]
            # sigma >= 3: within [0.75, 1.35] x paper.  sigma = 1: the gradients of the literal
            # per-tile psi(P)/psi(dS) reading (A11) sit up to ~3.7x above the paper.
            lo, hi = (0.75, 1.35) if (name == "o" or s >= 3) else (0.75, 4.5)
            assert lo * paper <= got <= hi * paper, (s, name, got, paper)
    # sigma = 10: dQ/dK cosine collapses below 0.9 (paper 0.78)
    assert res[10.0]["dq"][0] < 0.9 and res[10.0]["dk"][0] < 0.9


def test_k_smoothing_matters_on_outlier_k(orc):
    """K-smoothing is what keeps INT8 QK^T accurate under channel outliers:
    with outlier-injected K the quantised dQ error vs FPA must drop >= 2x when it is on."""
    q, k, v, do = (f64(t).reshape(2, 512, 64) for t in make_inputs(1, 2, 512, 64, "outlier_k", seed=12))
    on = _fidelity(orc, q, k, v, do, causal=True, k_smooth=True)
    off = _fidelity(orc, q, k, v, do, causal=True, k_smooth=False)
    assert off["dq"][1] > 2.0 * on["dq"][1]
    assert on["o"][1] < 0.05


def test_q_smoothing_bias_pathways(orc):
    """Q-smoothing with the bias added back and dK_bias keeps the quantised
    method close to FPA even with large Q channel offsets; dropping either term would not."""
    q, k, v, do = (f64(t).reshape(2, 256, 64) for t in make_inputs(1, 2, 256, 64, "outlier_kq", seed=13))
    q = q + 20.0                           # a large block mean makes mu_Q matter
    res = _fidelity(orc, q, k, v, do, causal=True, k_smooth=True, q_smooth=True)
    assert res["o"][1] < 0.06
    assert res["dk"][1] < 0.15 and res["dq"][1] < 0.15


def test_bwd_tile_dumps(orc):
    """The tile dumps (Tier-C and fidelity reports) are Alg. 2's own intermediates:
    - quant-off dS equals FPA's dS = P o (dP - delta) element-wise, so its
      rows sum to 0 (sum_n P (dP - delta) = delta - delta);
    - quantised mode: each dumped dS^ tile is psi of the dumped pre-psi dS tile (line 9, A4, A11):
      max|dS^| = 127 for a nonzero tile and |dS - dS^ s_dS| <= s_dS/2;
    - psi(P) per tile (line 6): P^ in [0, 127], 127 attained, s_P = max P / 127 with P = exp(S - L)
      <= 1, and tiles a causal run skips (above the diagonal) stay empty."""
    q, k, v, do = (f64(t).reshape(1, 384, 64) for t in make_inputs(1, 1, 384, 64, "gauss", seed=21, sigma=2.0))
    exact = orc.fwd(q, k, v, causal=True, quant=False)
    be = orc.bwd(q, k, v, exact["o"], do, exact["lse"], causal=True, quant=False, tiles=True)
    ref = orc.fpa(q, k, v, do, causal=True, intermediates=True)
    np.testing.assert_allclose(be["ds"], ref["dS"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(be["ds"].sum(2), 0.0, rtol=0, atol=1e-12)

    f = orc.fwd(q, k, v, causal=True)
    b = orc.bwd(q, k, v, f["o"], do, f["lse"], causal=True, tiles=True)
    for i in range(3):
        for j in range(3):
            blk = np.s_[0, i * 128:(i + 1) * 128, j * 128:(j + 1) * 128]
            ds, ds8, sds = b["ds"][blk], b["ds8"][blk].astype(np.float64), float(b["sds"][0, i, j])
            p8, sp = b["p8"][blk].astype(int), float(b["sp"][0, i, j])
            if j > i:
                assert sds == 0.0 and sp == 0.0 and not ds8.any() and not p8.any()
                continue
            assert np.abs(ds8).max() == 127
            assert sds == pytest.approx(np.abs(ds).max() / 127.0, rel=2 ** -23)
            assert np.abs(ds - ds8 * sds).max() <= sds * (0.5 + 2 ** -15)
            assert p8.min() >= 0 and p8.max() == 127 and 0.0 < sp <= 1.0 / 127.0 * (1 + 2 ** -23)


def test_p_u8_variant(orc):
    """Unsigned P^ (readings A2/A10 with 255 levels): P~ >= 0, so the
    per-token scale s_P = rowmax(P~)/255 (Alg. 1 line 9 with 255 for 127) and psi(P) over the
    backward tile (line 6) use 0..255.  Pins: the S:150 example at 255 levels; every tile's P^
    attains 255 with s_P = max P / 255; halving the rounding step lowers O's and dV's error
    against FPA (both carry P^'s rounding noise) while dQ/dK (dominated by dS) barely move."""
    q, sp = orc.psi_token_row(np.array([1.0, 0.5]), 0.0, pmax=255)
    assert list(q) == [255, 128] and sp == pytest.approx(1.0 / 255.0, rel=1e-15)
    errs = {}
    for u8 in (False, True):
        acc = {"o": [], "dv": [], "dq": []}
        for seed, recipe in ((31, "gauss"), (32, "qknorm")):
            q, k, v, do = (f64(t).reshape(2, 512, 64) for t in make_inputs(1, 2, 512, 64, recipe, seed=seed))
            ref = orc.fpa(q, k, v, do, causal=True)
            f = orc.fwd(q, k, v, causal=True, p_u8=u8)
            b = orc.bwd(q, k, v, f["o"], do, f["lse"], causal=True, p_u8=u8, tiles=True)
            acc["o"].append(rel_l2(ref["o"], f["o"]))
            acc["dv"].append(rel_l2(ref["dv"], b["dv"]))
            acc["dq"].append(rel_l2(ref["dq"], b["dq"]))
            if u8:
                for i in range(4):
                    p8 = b["p8"][0, i * 128:(i + 1) * 128, i * 128:(i + 1) * 128]
                    assert p8.max() == 255
                    assert float(b["sp"][0, i, i]) <= 1.0 / 255.0 * (1 + 2 ** -23)
        errs[u8] = {k_: float(np.mean(v_)) for k_, v_ in acc.items()}
    assert errs[True]["o"] < 0.95 * errs[False]["o"], errs
    assert errs[True]["dv"] < 0.7 * errs[False]["dv"], errs
    assert abs(errs[True]["dq"] - errs[False]["dq"]) < 0.25 * errs[False]["dq"], errs


# --------------------------------------------------------------------------- QK-norm
def test_qknorm_forward_closed_forms(orc):
    """RMSNorm (eps 1e-6 P:405; readings A24, A25): a constant row a gives
    rstd = 1/sqrt(a^2 + eps); the unrounded output has mean square m/(m + eps) per row; the
    output is bf16-valued and within half a bf16 ulp of x rstd gamma."""
    qn = orc.qknorm
    a = np.full((1, 64), 3.0)
    y, r = qn.forward(a, np.ones(64), eps=1e-6)
    assert float(r[0]) == np.float32(1.0 / math.sqrt(9.0 + 1e-6))
    rng = np.random.default_rng(40)
    x = torch.from_numpy(rng.standard_normal((4, 256, 128)) * 5).to(torch.bfloat16).double().numpy()
    g = rng.uniform(0.5, 2.0, 128).astype(np.float32)
    y0, r = qn.forward(x, np.ones(128), round_output=False)
    m = (x * x).mean(-1)
    np.testing.assert_allclose((y0 * y0).mean(-1), m / (m + 1e-6), rtol=1e-6)
    y, _ = qn.forward(x, g)
    exact = x * r[..., None].astype(np.float64) * g
    assert np.all(np.abs(y - exact) <= np.abs(exact) * 2.0 ** -8 * 1.0001)
    assert np.array_equal(y, torch.from_numpy(y).to(torch.bfloat16).double().numpy())


def test_qknorm_backward_finite_differences(orc):
    """dx and dgamma of y = x rstd(x) gamma (reading A26) against central finite differences of
    L = sum(w o y) in double (rstd exact, unrounded output)."""
    qn = orc.qknorm
    rng = np.random.default_rng(41)
    x = rng.standard_normal((3, 16))
    g = rng.uniform(0.5, 2.0, 16)
    w = rng.standard_normal((3, 16))
    eps = 1e-3

    def loss(xx, gg):
        r = 1.0 / np.sqrt((xx * xx).mean(-1, keepdims=True) + eps)
        return float((w * xx * r * gg).sum())
    r = 1.0 / np.sqrt((x * x).mean(-1) + eps)
    dx, dg = qn.backward(x, g, r, w)
    h = 1e-6
    fdx = np.zeros_like(x)
    for idx in np.ndindex(*x.shape):
        e = np.zeros_like(x)
        e[idx] = h
        fdx[idx] = (loss(x + e, g) - loss(x - e, g)) / (2 * h)
    fdg = np.array([(loss(x, g + h * np.eye(16)[c]) - loss(x, g - h * np.eye(16)[c])) / (2 * h) for c in range(16)])
    assert rel_l2(fdx, dx) < 1e-7 and rel_l2(fdg, dg) < 1e-7


def test_p_col_variant(orc):
    """Backward psi(P) per key column of the tile (ORC_P_COL, the dV half of SURVEY.md 8(f) NEXT-2):
    every key column of every processed tile attains the full 0..127 range, the forward is untouched,
    and dV's error against FPA drops well below the per-tile reading's (A11) at sigma = 1, the
    Table 1 row where the per-tile psi(P) leaves dV ~3.5x above the paper."""
    q, k, v, do = (f64(t).reshape(1, 512, 64) for t in make_inputs(1, 1, 512, 64, "gauss", seed=33, sigma=1.0))
    ref = orc.fpa(q, k, v, do)
    f = orc.fwd(q, k, v)
    errs = {}
    for pc in (False, True):
        b = orc.bwd(q, k, v, f["o"], do, f["lse"], p_col=pc, tiles=True)
        errs[pc] = {n: rel_l2(ref[n], b[n]) for n in ("dq", "dk", "dv")}
        if pc:
            p8 = b["p8"][0].reshape(4, 128, 4, 128)
            assert np.all(p8.max(axis=1) == 127)  # max over the queries of each key column, every tile
    assert errs[True]["dv"] < 0.5 * errs[False]["dv"], errs
    assert errs[True]["dq"] == errs[False]["dq"] and errs[True]["dk"] == errs[False]["dk"], errs


def test_ds_fine_variant(orc):
    """psi(dS) per query row for dQ and per key column for dK (ORC_DS_FINE, the dS half of SURVEY.md
    8(f) NEXT-2: the paper's named future work on the dS path): quant-off is unaffected;
    at Table 1's sigma = 1 dQ and dK get well below the per-tile reading's error (A11), with dV and O
    untouched; with Q-smoothing the dK bias pathway still holds."""
    q, k, v, do = (f64(t).reshape(1, 512, 64) for t in make_inputs(1, 1, 512, 64, "gauss", seed=34, sigma=1.0))
    ref = orc.fpa(q, k, v, do)
    f = orc.fwd(q, k, v)
    e = {}
    for fine in (False, True):
        b = orc.bwd(q, k, v, f["o"], do, f["lse"], ds_fine=fine)
        e[fine] = {n: rel_l2(ref[n], b[n]) for n in ("dq", "dk", "dv")}
    assert e[True]["dq"] < 0.6 * e[False]["dq"] and e[True]["dk"] < 0.6 * e[False]["dk"], e
    assert e[True]["dv"] == e[False]["dv"], e
    ex = orc.fwd(q, k, v, quant=False)
    b0 = orc.bwd(q, k, v, ex["o"], do, ex["lse"], quant=False)
    b1 = orc.bwd(q, k, v, ex["o"], do, ex["lse"], quant=False, ds_fine=True)
    assert np.array_equal(b0["dq"], b1["dq"]) and np.array_equal(b0["dk"], b1["dk"])
    q2, k2, v2, do2 = (f64(t).reshape(2, 256, 64) for t in make_inputs(1, 2, 256, 64, "outlier_kq", seed=13))
    q2 = q2 + 20.0
    ref2 = orc.fpa(q2, k2, v2, do2, causal=True)
    f2 = orc.fwd(q2, k2, v2, causal=True, q_smooth=True)
    b2 = orc.bwd(q2, k2, v2, f2["o"], do2, f2["lse"], causal=True, q_smooth=True, ds_fine=True)
    assert rel_l2(ref2["dk"], b2["dk"]) < 0.15 and rel_l2(ref2["dq"], b2["dq"]) < 0.15


def _block_scaled_inputs(N=384, d=64, seed=41):
    """Q, K, V, dO whose 128-row blocks differ in scale by 8x and 64x, in a different order for each tensor,
    so every block's psi scale differs from every other block's by >= 8x (fp32-exact values)."""
    rng = np.random.default_rng(seed)
    T = N // 128
    facs = {"q": (1.0, 8.0, 64.0), "k": (64.0, 1.0, 8.0), "v": (8.0, 64.0, 1.0), "do": (1.0, 64.0, 8.0)}
    base = {"q": 0.02, "k": 0.02, "v": 1.0, "do": 1.0}
    out = {}
    for name in ("q", "k", "v", "do"):
        x = rng.standard_normal((1, N, d))
        for t in range(T):
            x[:, t * 128:(t + 1) * 128] *= base[name] * facs[name][t % 3]
        out[name] = x.astype(np.float32).astype(np.float64)
    return out["q"], out["k"], out["v"], out["do"]


@pytest.mark.parametrize("causal", [False, True])
def test_block_scale_bookkeeping(orc, causal):
    """Per-block scales (Alg. 1 lines 3, 7, 10; Alg. 2 lines 6-11): with Q, K, V, dO
    blocks whose scales differ 8-64x, the quantised oracle stays as close to FPA as with uniform blocks
    (rel-L2 < 0.08 for O, dQ, dK, dV).  A tile that used the wrong block's s_Q, s_K, s_V or s_dO would be
    off by >= 8x on that tile, which is >= 0.5 rel-L2 on the affected output (checked by mutation, see the
    commit that added this pin)."""
    q, k, v, do = _block_scaled_inputs()
    res = _fidelity(orc, q, k, v, do, causal=causal, k_smooth=False)
    for name in ("o", "dq", "dk", "dv"):
        assert res[name][1] < 0.08, (name, res)


def test_block_selection_is_the_full_run(orc):
    """The sampled-output mode (q_blocks / k_blocks) used for full-size parity checks runs the same
    tiles in the same order as the full run: its selected rows are bitwise those of the full run."""
    q, k, v, do = (f64(t).reshape(2, 512, 64) for t in make_inputs(1, 2, 512, 64, "outlier_kq", seed=17))
    for causal, qs in ((True, False), (False, True)):
        kw = dict(causal=causal, k_smooth=True, q_smooth=qs)
        f = orc.fwd(q, k, v, **kw)
        fs = orc.fwd(q, k, v, q_blocks=[0, 3], **kw)
        for blk in (0, 3):
            rows = slice(blk * 128, (blk + 1) * 128)
            np.testing.assert_array_equal(fs["o"][:, rows], f["o"][:, rows])
            np.testing.assert_array_equal(fs["lse"][:, rows], f["lse"][:, rows])
        assert not fs["o"][:, 128:384].any()
        b = orc.bwd(q, k, v, f["o"], do, f["lse"], **kw)
        bs = orc.bwd(q, k, v, f["o"], do, f["lse"], q_blocks=[1, 3], k_blocks=[0, 2], **kw)
        for name, blocks in (("dq", (1, 3)), ("dk", (0, 2)), ("dv", (0, 2))):
            for blk in blocks:
                rows = slice(blk * 128, (blk + 1) * 128)
                np.testing.assert_array_equal(bs[name][:, rows], b[name][:, rows])
        assert not bs["dq"][:, :128].any() and not bs["dk"][:, 128:256].any()
        np.testing.assert_array_equal(bs["delta"], b["delta"])


def test_forward_tile_dump(orc):
    """The forward dump (Tier C of K2) is Alg. 1 line 9's per-token P^: every processed row of a
    tile has P^ in [0, 127] with 127 attained at the row's max, s_P = e^{rowmax - m_ij} / 127 <= 1/127
    (m_ij >= rowmax); causal tiles above the diagonal stay empty; the dump does not change O."""
    q, k, v, _ = (f64(t).reshape(1, 384, 64) for t in make_inputs(1, 1, 384, 64, "gauss", seed=23, sigma=1.5))
    f = orc.fwd(q, k, v, causal=True, tiles=True)
    f0 = orc.fwd(q, k, v, causal=True)
    np.testing.assert_array_equal(f["o"], f0["o"])
    p8, sp = f["p8"][0], f["sp"][0]
    assert p8.max() <= 127
    for i in range(3):
        for j in range(3):
            tile = p8[i * 128:(i + 1) * 128, j * 128:(j + 1) * 128]
            if j > i:
                assert not tile.any()
                continue
            rows_max = tile.max(axis=1)
            assert (rows_max == 127).all()
            assert (sp[i * 128:(i + 1) * 128, j] <= 1.0 / 127.0 + 1e-15).all()
    assert (sp[:, 0] > 0).all()


# --------------------------------------------------------------------------- precision policy
def _policy_inputs(N=256, d=64, seed=51):
    """fp32 inputs (so that the fp16-emulated tag rounds something; bf16 values are fp16-exact)."""
    q, k, v, do = (f64(t).reshape(N, d) for t in make_inputs(1, 1, N, d, "qknorm", seed=seed, dtype=torch.float32))
    return q, k, v, do


@pytest.mark.parametrize("causal", [False, True])
def test_policy_exact_is_fpa(orc, causal):
    """The pseudo-quantisation harness with every site exact is full-precision attention: it matches the
    C oracle's independent FPA (oracle_fpa) in every intermediate."""
    q, k, v, do = _policy_inputs()
    got = orc.policy.attention(q, k, v, do, orc.policy.EXACT, causal=causal, k_smooth=False)
    ref = orc.fpa(q[None], k[None], v[None], do[None], causal=causal, intermediates=True)
    for a, b in (("O", "o"), ("dQ", "dq"), ("dK", "dk"), ("dV", "dv"), ("P", "P"), ("dP", "dP"), ("dS", "dS"),
                 ("delta", "delta"), ("L", "lse")):
        np.testing.assert_allclose(got[a], ref[b][0], rtol=1e-9, atol=1e-12, err_msg=a)


def test_policy_site_dependencies(orc):
    """Each site quantised alone perturbs exactly the quantities downstream of its MatMul in Alg. 1/2's
    dataflow (a mis-wired operand fails here): qk -> everything but dP; pv -> O, delta, dS, dQ, dK;
    dv -> dV only; dp (fp16) -> dP, dS, dQ, dK; dq -> dQ only; dk -> dK only.  K-smoothing alone is exact
    (a per-row constant shift of S)."""
    q, k, v, do = _policy_inputs()
    P = orc.policy
    ref = P.attention(q, k, v, do, P.EXACT, k_smooth=False)
    smoothed = P.attention(q, k, v, do, P.EXACT, k_smooth=True)
    for n in ("O", "dQ", "dK", "dV"):
        np.testing.assert_allclose(smoothed[n], ref[n], rtol=1e-9, atol=1e-12)
    names = ("P", "O", "delta", "dP", "dS", "dQ", "dK", "dV")
    expect = {"qk": {"P", "O", "delta", "dS", "dQ", "dK", "dV"}, "pv": {"O", "delta", "dS", "dQ", "dK"},
              "dv": {"dV"}, "dp": {"dP", "dS", "dQ", "dK"}, "dq": {"dQ"}, "dk": {"dK"}}
    for site, changed in expect.items():
        pol = dict(P.EXACT)
        pol[site] = "fp16-emulated" if site == "dp" else P.SAGEBWD[site]
        got = P.attention(q, k, v, do, pol, k_smooth=False)
        for n in names:
            err = P.rel_l2(ref[n], got[n])
            if n in changed:
                assert err > 1e-6, (site, n, err)
            else:
                assert err < 1e-12, (site, n, err)


def test_policy_sagebwd_tracks_tiled_oracle(orc):
    """With SageBwd's policy the harness reproduces the tiled quantised oracle's error against FPA within
    25% for O, dQ, dK, dV (they differ only in the per-token P^ reference max, reading A10).  Table 2's
    finding: the dS operand after psi carries far more error than O, and dQ / dK get
    most of their error from quantising dS at their own sites (the single-site ablation), while dP is
    exact (its BF16 operands are the I/O values, reading A9)."""
    q, k, v, do = _policy_inputs(N=512, d=64, seed=52)
    comp = orc.policy.component_errors(q, k, v, do, causal=True)
    ref = orc.fpa(q[None], k[None], v[None], do[None], causal=True)
    f = orc.fwd(q[None], k[None], v[None], causal=True)
    b = orc.bwd(q[None], k[None], v[None], f["o"], do[None], f["lse"], causal=True)
    tiled = {"O": rel_l2(ref["o"], f["o"]), "dQ": rel_l2(ref["dq"], b["dq"]), "dK": rel_l2(ref["dk"], b["dk"]),
             "dV": rel_l2(ref["dv"], b["dv"])}
    for n, t in tiled.items():
        assert abs(comp[n] - t) <= 0.25 * t, (n, comp[n], t)
    assert comp["dS_post_psi"] > 3 * comp["O"] and comp["dP"] == 0.0
    abl = orc.policy.site_ablation(q, k, v, do, causal=True)
    assert abl["dq"]["dQ"] >= 0.8 * comp["dQ"] and abl["dk"]["dK"] >= 0.8 * comp["dK"], abl


# --------------------------------------------------------------------------- FP8 P^V^ variant (NEXT-4)
def test_e4m3_rounding_matches_torch(orc):
    """oracle.e4m3 is round-to-nearest-even into FP8 E4M3 (3 mantissa bits, bias 7, subnormals at 2^-9):
    pinned against torch's float8_e4m3fn conversion on every E4M3 value, every midpoint between neighbours
    (ties to even) and random values in [-448, 448]."""
    grid = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float()
    vals = grid[torch.isfinite(grid)].double().unique().numpy()
    mids = (vals[1:] + vals[:-1]) / 2
    rng = np.random.default_rng(3)
    rand = np.concatenate([rng.uniform(-448, 448, 4000), rng.uniform(-1, 1, 4000) * 2.0 ** rng.integers(-12, 0, 4000)])
    for x in np.concatenate([vals, mids, rand]):
        want = torch.tensor([x], dtype=torch.float64).to(torch.float8_e4m3fn).double().item()
        assert orc.e4m3(x) == want, (x, orc.e4m3(x), want)
    assert orc.e4m3(460.0) == 448.0 and orc.e4m3(-1e9) == -448.0   # saturation (satfinite)


def test_pv_fp8_mode(orc):
    """ORC_PV_FP8 (Alg. 1 lines 9-10 with E4M3 instead of INT8 P^ and V^): V^ per block is psi_block_e4m3
    (|V^| <= 448, 448 attained, scale = amax/448), L is unchanged (l is built from the unquantised P~,
    reading A10), the backward is untouched, and O's error against FPA is that of E4M3's 3-bit mantissa:
    larger than the INT8 path's (127 levels per block / per token) by 2-4x on Gaussian V, and below 0.06."""
    q, k, v, do = (f64(t).reshape(2, 384, 64) for t in make_inputs(1, 2, 384, 64, "qknorm", seed=61))
    fpa = orc.fpa(q, k, v, causal=True)
    f8 = orc.fwd(q, k, v, causal=True, pv_fp8=True)
    f = orc.fwd(q, k, v, causal=True)
    np.testing.assert_array_equal(f8["lse"], f["lse"])
    for t in range(3):
        vq, sv = orc.psi_block_e4m3(v[0, t * 128:(t + 1) * 128])
        assert np.abs(vq).max() == 448.0 and sv == np.float32(np.abs(v[0, t * 128:(t + 1) * 128]).max() / np.float32(448))
        assert f8["sv"][0, t] == np.float32(sv)
    e8, e = rel_l2(fpa["o"], f8["o"]), rel_l2(fpa["o"], f["o"])
    assert 1.5 * e <= e8 <= 4.0 * e and e8 < 0.06, (e8, e)
