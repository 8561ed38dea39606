"""Randomised GPU parity: seeded draws over the whole option space (N including ragged lengths, d, causal,
K / Q smoothing, B and H, the flag variants, the softmax scale) against the oracle's matching mode, at the
north-star tolerance.  Complements the hand-picked cases of test_gpu.py / test_gpu_ragged.py: a combination
nobody thought to list still gets checked."""
import numpy as np
import pytest
import torch

import oracle
from paper_2603_02170_b200 import sage
from paper_2603_02170_b200.inputs import make_inputs
from tests.metrics import f64, round_bf16
from tests.test_gpu import _assert_ok, _compare

pytestmark = pytest.mark.gpu

VARIANTS = ["none", "none", "none", "p_u8", "pv_fp8", "p_colscale", "fine_bwd", "deterministic", "fp32_out"]
RECIPES = ["gauss", "qknorm", "outlier_k", "outlier_kq"]


def _draw(seed):
    rng = np.random.default_rng(seed)
    N = int(rng.choice([int(rng.integers(1, 1100)), 128 * int(rng.integers(1, 9))]))
    d = int(rng.choice([64, 128]))
    B, H = int(rng.integers(1, 3)), int(rng.integers(1, 3))
    causal, ks, qs = bool(rng.integers(2)), bool(rng.integers(2)), bool(rng.integers(2))
    variant = str(rng.choice(VARIANTS))
    if variant == "deterministic" and not causal and -(-N // 128) > 100:
        variant = "none"
    tau = None if rng.integers(2) else float(rng.uniform(0.03, 0.3))
    recipe = str(rng.choice(RECIPES))
    if recipe.startswith("outlier"):
        # outlier K without K-smoothing is the method's documented failure regime: its own error
        # against FPA is ~34% there, and P^ rounding ties (Tier C) then move dQ by ~2e-3 against the oracle
        # (measured with SAGE_P_U8: 2.1e-3) -- the output tolerance is not meaningful there
        ks = True
    return dict(N=N, d=d, B=B, H=H, causal=causal, ks=ks, qs=qs, variant=variant, tau=tau, recipe=recipe)


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    assert torch.cuda.is_available() and torch.cuda.get_device_capability() == (10, 0)
    sage.lib()
    oracle.build()


@pytest.mark.parametrize("seed", range(24))
def test_random_parity(seed):
    c = _draw(9000 + seed)
    B, H, N, d = c["B"], c["H"], c["N"], c["d"]
    q, k, v, do = make_inputs(B, H, N, d, c["recipe"], seed=3000 + seed)
    dev = "cuda"
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    var = c["variant"]
    kw = {} if var == "none" else {var: True}
    o, lse, ctx = sage.forward(qd, kd, vd, causal=c["causal"], k_smooth=c["ks"], q_smooth=c["qs"],
                               softmax_scale=c["tau"], **kw)
    dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
    torch.cuda.synchronize()
    heads = list(range(B * H))
    sel = lambda t: f64(t).reshape(B * H, N, d)
    okw = dict(causal=c["causal"], k_smooth=c["ks"], q_smooth=c["qs"], tau=c["tau"])
    f = oracle.fwd(sel(q), sel(k), sel(v), p_u8=var == "p_u8", pv_fp8=var == "pv_fp8", **okw)
    rnd = (lambda x: x) if var == "fp32_out" else round_bf16
    b = oracle.bwd(sel(q), sel(k), sel(v), rnd(f["o"]), sel(do), f["lse"], p_u8=var == "p_u8",
                   p_col=var in ("p_colscale", "fine_bwd"), ds_fine=var == "fine_bwd", **okw)
    gpu = dict(o=o, lse=lse, dq=dq, dk=dk, dv=dv)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d, out_round=rnd), c)


@pytest.mark.parametrize("B,H,d,causal", [(1, 5, 64, True), (3, 1, 128, True), (1, 7, 128, False)])
def test_head_counts_around_the_cta_groups(B, H, d, causal):
    """K2 / K4 order their CTAs in groups of 4 heads (the last group short): head counts that leave a partial
    group must still cover every (head, block) once."""
    from tests.test_gpu import _oracle, _run
    N = 384
    q, k, v, do = make_inputs(B, H, N, d, "qknorm", seed=3100 + B * H + d)
    gpu = _run(q, k, v, do, causal, True, False)
    heads = list(range(B * H))
    f, b = _oracle(q, k, v, do, heads, causal, True, False)
    _assert_ok(_compare(gpu, f, b, heads, B, H, N, d), (B, H, d, causal))
