"""Seeded synthetic inputs shaped like the paper's workloads.

This module holds NO arithmetic of the method: it only draws Q, K, V, dO.  It is
the one piece shared by the CUDA-path tests, the oracle tests, smoke() and
bench.py (task rule: "only the seeded input generators serve both").

Recipes:
  gauss(sigma)   Q, K ~ N(0, sigma^2); V, dO ~ N(0, 1)              (Table 1)
  qknorm(gamma)  X ~ N(0,1) diag(exp(N(0, 0.5^2))) + +-10 offsets on 4 channels,
                 Q = RMSNorm(X_q) gamma, K = RMSNorm(X_k) gamma, eps = 1e-6
  outlier_k      K = N(0,1) + offset vector of +-15..20 on 4 channels (q_outliers: Q +-6..8 on 4)
  noqknorm       the qknorm X without RMSNorm, scaled to sigma = 3
Seeds: head (b, h) of a run with base seed s uses torch.Generator().manual_seed(s + global_head),
so data is identical for every GPU count and for the oracle.
"""
from dataclasses import dataclass

import torch


@dataclass(frozen=True)
class Config:
    name: str
    batch: int
    heads: int
    seqlen: int
    head_dim: int
    causal: bool
    k_smooth: bool
    q_smooth: bool
    recipe: str
    seed: int


# BASELINE.json "configs", in order (C1..C5).
CONFIGS = {
    "C1": Config("C1", 1, 2, 128, 64, True, True, False, "outlier_k", 1000),
    "C2": Config("C2", 8, 16, 2048, 64, False, True, False, "qknorm", 2000),
    "C3": Config("C3", 4, 32, 4096, 128, True, True, True, "outlier_kq", 3000),
    "C4": Config("C4", 2, 32, 16384, 128, True, True, False, "qknorm", 4000),
    "C5": Config("C5", 16, 16, 8192, 128, True, True, False, "qknorm", 5000),
}
# The metric's sequence-length sweep ("TOPS ... at seqlen 1K-32K", BASELINE.json; SURVEY.md 8(d)
# C4-sweep): N in {1K, ..., 32K}, B = 32768 / N, H = 32, d = 128, causal, QK-normed inputs.
for _n in (1024, 2048, 4096, 8192, 16384, 32768):
    _name = f"S{_n // 1024}K"
    CONFIGS[_name] = Config(_name, 32768 // _n, 32, _n, 128, True, True, False, "qknorm", 6000 + _n // 1024)


def _rmsnorm(x, gamma, eps=1e-6):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps) * gamma


def _head(recipe, N, d, gen, sigma, gamma):
    """One head's (q, k, v, do) in float32."""
    def randn(*shape):
        return torch.randn(*shape, generator=gen, dtype=torch.float32)

    def offsets(lo, hi):
        ch = torch.randperm(d, generator=gen)[:4]
        mag = lo + (hi - lo) * torch.rand(4, generator=gen)
        sign = torch.where(torch.rand(4, generator=gen) < 0.5, -1.0, 1.0)
        off = torch.zeros(d)
        off[ch] = mag * sign
        return off

    def hetero():
        chan = torch.exp(0.5 * randn(d))
        return randn(N, d) * chan + offsets(10.0, 10.0)

    if recipe == "gauss":
        q, k = sigma * randn(N, d), sigma * randn(N, d)
    elif recipe == "qknorm":
        q, k = _rmsnorm(hetero(), gamma), _rmsnorm(hetero(), gamma)
    elif recipe == "noqknorm":
        xq, xk = hetero(), hetero()
        q, k = 3.0 * xq / xq.std(), 3.0 * xk / xk.std()
    elif recipe in ("outlier_k", "outlier_kq"):
        q = randn(N, d)
        k = randn(N, d) + offsets(15.0, 20.0)
        if recipe == "outlier_kq":
            q = q + offsets(6.0, 8.0)
    else:
        raise ValueError(recipe)
    v, do = randn(N, d), randn(N, d)
    return q, k, v, do


def make_inputs(batch, heads, seqlen, head_dim, recipe="qknorm", seed=0, head_offset=0,
                sigma=1.0, gamma=1.0, dtype=torch.bfloat16):
    """Return (q, k, v, do) as CPU tensors [B, H, N, d] of ``dtype``.

    Head (b, h) uses generator seed ``seed + head_offset + b*H + h``.
    """
    shape = (batch, heads, seqlen, head_dim)
    outs = [torch.empty(shape, dtype=dtype) for _ in range(4)]
    for b in range(batch):
        for h in range(heads):
            g = torch.Generator().manual_seed(seed + head_offset + b * heads + h)
            for t, x in zip(outs, _head(recipe, seqlen, head_dim, g, sigma, gamma)):
                t[b, h] = x.to(dtype)
    return tuple(outs)


def config_inputs(cfg: Config, head_offset=0, batch=None, dtype=torch.bfloat16):
    b = cfg.batch if batch is None else batch
    return make_inputs(b, cfg.heads, cfg.seqlen, cfg.head_dim, cfg.recipe, cfg.seed,
                       head_offset=head_offset, dtype=dtype)
