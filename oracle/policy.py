"""Per-MatMul precision policy: pseudo-quantised full-precision attention (TEST INFRASTRUCTURE ONLY).

The paper traces where SageBwd's error comes from (Table 2; method P:486-506) by "applying
the SageBwd INT8 quantize-dequantize scheme before each relevant matrix multiplication in a PyTorch
attention implementation" and comparing every intermediate (delta, P, dP, dS, O, dQ, dK, dV) against
full-precision attention (FPA).  SPEC.md's PrecisionPolicy names the six MatMul sites and
the tags this module implements:

  sites  qk  S  = tau Q K^T            (Alg. 1 line 7)     pv  O  = P V          (line 10)
         dv  dV = P^T dO               (Alg. 2 line 7)     dp  dP = dO V^T       (line 8)
         dq  dQ = tau dS K             (line 10)           dk  dK = tau dS^T Q   (line 11)
  tags   exact            no rounding (double)
         int8-per-block   psi over 128 x 128 tiles of an N x N operand, 128-row blocks of an N x d one
                          (scale = fl32(amax/127), q = RNE(fl32(x * fl32(127/amax))), readings A1-A4)
         int8-per-token   psi per row of each 128-column block (only for P at the pv site)
         fp16-emulated    operands rounded to fp16 (the paper's "FP16" dP)

SAGEBWD is the paper's own policy (qk, dv, dq, dk per block, pv per token) with dP exact: its operands are
the BF16 I/O values themselves and the MMA accumulates in FP32 (reading A9), so "FP16 dP" adds no rounding
to BF16 inputs; the fp16-emulated tag (rounding the operands to fp16) is there for FP32 inputs.  K-smoothing
 is applied before the qk site's quantisation, as SageBwd does.  Everything is materialised
N x N in float64; this is the paper's analysis harness, not the tiled online-softmax kernel (the oracle's
fwd / bwd are that), so the two differ by the per-token P^ reference max (tile row max here, the running
max there, reading A10).
"""
import numpy as np

SITES = ("qk", "pv", "dv", "dp", "dq", "dk")
TAGS = ("exact", "int8-per-block", "int8-per-token", "fp16-emulated")
SAGEBWD = dict(qk="int8-per-block", pv="int8-per-token", dv="int8-per-block", dp="exact",
               dq="int8-per-block", dk="int8-per-block")
EXACT = {s: "exact" for s in SITES}
BLK = 128


def _psi(x):
    """psi of one block (readings A1-A4): the dequantised values q * scale."""
    f32 = np.float32
    amax = f32(np.abs(x).max()) if x.size else f32(0)
    if amax == 0:
        return np.zeros_like(x)
    scale = f32(amax / f32(127))
    inv = f32(f32(127) / amax)
    q = np.clip(np.rint((x.astype(f32) * inv).astype(np.float64)), -127, 127)  # rint: round half to even
    return q * np.float64(scale)


def quant(x, tag, rows_only=False):
    """Dequantised x under `tag`.  x: [N, M] float64.  rows_only: an N x d operand (blocks of 128 rows)."""
    if tag == "exact":
        return x.copy()
    if tag == "fp16-emulated":
        return x.astype(np.float16).astype(np.float64)
    out = np.empty_like(x)
    N, M = x.shape
    cb = M if rows_only else BLK
    for r0 in range(0, N, BLK):
        for c0 in range(0, M, cb):
            blk = x[r0:r0 + BLK, c0:c0 + cb]
            if tag == "int8-per-block":
                out[r0:r0 + BLK, c0:c0 + cb] = _psi(blk)
            elif tag == "int8-per-token":
                out[r0:r0 + BLK, c0:c0 + cb] = np.stack([_psi(row) for row in blk])
            else:
                raise ValueError(tag)
    return out


def _rows_tag(tag):
    """The tag of the N x d operand at a site whose N x N operand has `tag` (per token -> per block)."""
    return "int8-per-block" if tag == "int8-per-token" else tag


def attention(q, k, v, do, policy=SAGEBWD, causal=False, k_smooth=True, tau=None):
    """One head, every intermediate of Alg. 1/2's dataflow with each MatMul's operands under `policy`.
    q, k, v, do: [N, d] float64.  Returns dict(S, P, L, O, delta, dP, dS, dQ, dK, dV)."""
    for s in SITES:
        if policy[s] not in TAGS:
            raise ValueError((s, policy[s]))
    if policy["qk"] == "int8-per-token" or any(policy[s] == "int8-per-token" for s in SITES if s != "pv"):
        raise ValueError("int8-per-token is only valid at the pv site (S:208)")
    N, d = q.shape
    tau = 1.0 / np.sqrt(d) if tau is None else tau
    ks = k - k.mean(axis=0) if k_smooth else k          # K-smoothing: a per-row constant shift of S
    S = tau * quant(q, policy["qk"], True) @ quant(ks, policy["qk"], True).T
    if causal:
        S = np.where(np.tril(np.ones((N, N), bool)), S, -np.inf)
    m = S.max(axis=1, keepdims=True)
    E = np.exp(S - m)
    l = E.sum(axis=1, keepdims=True)
    P = E / l
    L = (m + np.log(l))[:, 0]
    # pv: P per token (row of each 128-column block) and V per 128-row block; P is in [0, 1]
    O = quant(P, policy["pv"]) @ quant(v, _rows_tag(policy["pv"]), True)
    delta = (do * O).sum(axis=1)
    dV = quant(P, policy["dv"]).T @ quant(do, policy["dv"], True)
    dP = quant(do, policy["dp"], True) @ quant(v, policy["dp"], True).T
    dS = P * (dP - delta[:, None])
    dS_q = quant(dS, policy["dq"])  # the dQ site's dS operand ("dS post-psi")
    # dQ uses the smoothed K (Alg. 2 line 10 takes K^ = psi(K_sm)); dS K_sm = dS K for exact dS
    dQ = tau * dS_q @ quant(ks, policy["dq"], True)
    dK = tau * quant(dS, policy["dk"]).T @ quant(q, policy["dk"], True)
    return dict(S=S, P=P, L=L, O=O, delta=delta, dP=dP, dS=dS, dS_q=dS_q, dQ=dQ, dK=dK, dV=dV)


def rel_l2(ref, x):
    ref, x = np.asarray(ref, np.float64).ravel(), np.asarray(x, np.float64).ravel()
    ok = np.isfinite(ref)
    return float(np.linalg.norm(ref[ok] - x[ok]) / np.linalg.norm(ref[ok]))


def component_errors(q, k, v, do, policy=SAGEBWD, causal=False, k_smooth=True):
    """Table 2's rows: rel-L2 of delta, P, dP, dS (before and after the dQ site's psi), O, dQ,
    dK, dV under `policy` against FPA."""
    ref = attention(q, k, v, do, EXACT, causal, k_smooth=False)
    got = attention(q, k, v, do, policy, causal, k_smooth)
    out = {n: rel_l2(ref[n], got[n]) for n in ("delta", "P", "dP", "dS", "O", "dQ", "dK", "dV")}
    out["dS_post_psi"] = rel_l2(ref["dS"], got["dS_q"])
    return out


def site_ablation(q, k, v, do, causal=False, k_smooth=True):
    """Each MatMul site quantised alone (SageBwd's tag there, exact elsewhere), plus the full policy:
    which site's quantisation produces which component's error (the Table 2 analysis)."""
    rows = {}
    for s in SITES:
        pol = dict(EXACT)
        pol[s] = SAGEBWD[s]
        rows[s] = component_errors(q, k, v, do, pol, causal, k_smooth)
    rows["all"] = component_errors(q, k, v, do, SAGEBWD, causal, k_smooth)
    return rows
