"""QK-norm, the step before the SageBwd path (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

PAPER.md P:212-234 (Sec. 4.1 "Stabilizing Outliers with QK-Norm"): RMS normalisation of every
token of Q and K with a learned scale vector gamma, eps = 1e-6 ("a norm
epsilon of 1e-6"), BF16 mixed precision.  Readings (A24-A26):

  A24  rstd[r] = fl32(1 / sqrt(sum_c x[r,c]^2 / d + eps)), eps the fp32 value: the sum of squares of the bf16 inputs
       in double (exact, hence order-free, unless a row's squares span > 30 binades), the
       division and square root in double, one rounding to fp32.
  A25  y[r,c] = bf16(fl32(fl32(x[r,c] * rstd[r]) * gamma[c])): the module output is BF16, as in
       an unfused BF16 mixed-precision pipeline; the SageBwd path then sees exactly these values.
  A26  backward: the attention gradient w.r.t. y is rounded to bf16 (the unfused module chain),
       then  g = dy o gamma,  xh = x rstd,  dx = rstd (g - xh mean_c(g o xh)),
       dgamma = sum over all rows of dy o xh  -- here in double.

Plain numpy, written from the definition; no code shared with the CUDA path.
"""
import numpy as np


def _bf16_round(x):
    """Round float32 values to bf16 (round-to-nearest-even), returned as float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def rstd(x, eps=1e-6):
    """A24: per-row reciprocal RMS of x [..., d] (bf16-valued), fp32."""
    x = np.asarray(x, dtype=np.float64)
    ss = (x * x).sum(-1)
    eps = float(np.float32(eps))   # the ABI carries eps as an fp32 value
    return (1.0 / np.sqrt(ss / x.shape[-1] + eps)).astype(np.float32)


def forward(x, gamma, eps=1e-6, round_output=True):
    """A25: y = RMSNorm(x) * gamma.  x [..., d] bf16-valued, gamma [d].  Returns (y, rstd)."""
    r = rstd(x, eps)
    xf = np.asarray(x, dtype=np.float32)
    g = np.asarray(gamma, dtype=np.float32)
    y = (xf * r[..., None]).astype(np.float32) * g          # two fp32 roundings
    y = y.astype(np.float32)
    if round_output:
        y = _bf16_round(y)
    return y.astype(np.float64), r


def backward(x, gamma, r, dy):
    """A26 in double: (dx, dgamma) for y = x * rstd * gamma with rstd = r (fp32 from forward)."""
    x = np.asarray(x, dtype=np.float64)
    g = np.asarray(gamma, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)[..., None]
    dy = np.asarray(dy, dtype=np.float64)
    xh = x * r
    gd = dy * g
    dx = r * (gd - xh * (gd * xh).mean(-1, keepdims=True))
    dgamma = (dy * xh).reshape(-1, x.shape[-1]).sum(0)
    return dx, dgamma
