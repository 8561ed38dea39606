"""ctypes front-end of ``liboracle.so`` (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Arrays are numpy, [BH, N, d] float64 (inputs must hold bf16/fp32-exact values
in quantised mode -- the oracle treats them as the FP32 numbers the kernels see).
"""
import ctypes
import os
import subprocess

import numpy as np

CAUSAL, K_SMOOTH, Q_SMOOTH, QUANT_OFF, P_U8, P_COL, DS_FINE, PV_FP8 = 1, 2, 4, 8, 16, 32, 64, 128

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sage_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force=False):
    """Compile liboracle.so with gcc: -O2 -ffp-contract=off (exact FP32 emulation), OpenMP."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-fPIC", "-shared", "-std=c11", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I, D = ctypes.c_int, ctypes.c_double
        _lib.oracle_fwd.argtypes = [I, I, I, I, I, D] + [P] * 14
        _lib.oracle_bwd.argtypes = [I, I, I, I, I, D] + [P] * 17
        _lib.oracle_fwd_sel.argtypes = [I, I, I, I, I, D] + [P] * 17
        _lib.oracle_bwd_sel.argtypes = [I, I, I, I, I, D] + [P] * 19
        _lib.oracle_fpa.argtypes = [I, I, I, I, D] + [P] * 13
        _lib.oracle_psi_block.argtypes = [P, I, I, P, P]
        _lib.oracle_psi_token_row.argtypes = [P, I, D, I, P]
        _lib.oracle_psi_token_row.restype = D
        _lib.oracle_set_threads.argtypes = [I]
        _lib.oracle_e4m3.argtypes = [D]
        _lib.oracle_e4m3.restype = D
        _lib.oracle_psi_block_e4m3.argtypes = [P, I, P, P]
        _lib.oracle_max_threads.restype = I
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n):
    _load().oracle_set_threads(int(n))


def max_threads():
    return _load().oracle_max_threads()


def psi_block(x, fp32_product=True):
    """psi over one block (reading A4).  Returns (int8 values, fp32 scale as float)."""
    x = _f64(x)
    q = np.zeros(x.shape, dtype=np.int8)
    s = np.zeros(1, dtype=np.float64)
    _load().oracle_psi_block(_p(x), x.size, int(fp32_product), _p(q), _p(s))
    return q, float(s[0])


def psi_token_row(pt, rm_minus_m, pmax=127):
    """Per-token P quantisation of one row (Alg. 1 line 9; pmax 255: the u8 variant).
    Returns (integer values, s_P)."""
    pt = _f64(pt)
    q = np.zeros(pt.shape, dtype=np.int16)
    sp = _load().oracle_psi_token_row(_p(pt), pt.size, float(rm_minus_m), int(pmax), _p(q))
    return q, sp


def e4m3(x):
    """FP8 E4M3 round-to-nearest-even with saturation at 448 (the PTX cvt.rn.satfinite conversion)."""
    return _load().oracle_e4m3(float(x))


def psi_block_e4m3(x):
    """psi into E4M3 over one block (the ORC_PV_FP8 V^): (e4m3 values, fp32 scale amax/448)."""
    x = _f64(x)
    q = np.zeros(x.shape, dtype=np.float64)
    s = np.zeros(1, dtype=np.float64)
    _load().oracle_psi_block_e4m3(_p(x), x.size, _p(q), _p(s))
    return q, float(s[0])


def _default_tau(d, tau):
    return 1.0 / np.sqrt(d) if tau is None else float(tau)


def _flags(causal, k_smooth, q_smooth, quant, p_u8, p_col=False, ds_fine=False, pv_fp8=False):
    return (CAUSAL if causal else 0) | (K_SMOOTH if k_smooth else 0) | (Q_SMOOTH if q_smooth else 0) | \
        (0 if quant else QUANT_OFF) | (P_U8 if p_u8 else 0) | (P_COL if p_col else 0) | (DS_FINE if ds_fine else 0) | \
        (PV_FP8 if pv_fp8 else 0)


def _sel(blocks, BH, T):
    """None, or a [BH][T] uint8 selection from a list of block indices (the same for every head)."""
    if blocks is None:
        return None
    m = np.zeros((BH, T), np.uint8)
    m[:, list(blocks)] = 1
    return m


def fwd(q, k, v, *, causal=False, k_smooth=True, q_smooth=False, quant=True, blk=128, tau=None, p_u8=False,
        q_blocks=None, tiles=False, pv_fp8=False):
    """Alg. 1 per head.  Returns dict with o, lse and the Tier-A intermediates.
    q_blocks: compute O and L only for these query blocks (other rows stay zero), with the same
    arithmetic as the full run (sampled checks at sizes the full oracle cannot finish).
    tiles=True also returns the per-token P^ of every processed tile (p8, [BH, N q, N kv] uint8; tile (i, j)
    at rows i*blk.., columns j*blk..; masked or skipped entries 0) and its row scale s_P (sp, [BH, N q, T]
    float64, Alg. 1 line 9).
    pv_fp8=True: P^ and V^ in FP8 E4M3 (ORC_PV_FP8); v8 is then left zero and the
    dumped p8 is zero (the E4M3 P^ is not an integer); sv holds the E4M3 block scales amax/448."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    BH, N, d = q.shape
    T = -(-N // blk)  # ceil: a ragged N has a short last block (reading A33)
    qsel = _sel(q_blocks, BH, T)
    flags = _flags(causal, k_smooth, q_smooth, quant, p_u8, pv_fp8=pv_fp8)
    out = dict(o=np.zeros((BH, N, d)), lse=np.zeros((BH, N)),
               mu_k=np.zeros((BH, d), np.float32), mu_q=np.zeros((BH, T, d), np.float32),
               bias=np.zeros((BH, T, N)),
               q8=np.zeros((BH, N, d), np.int8), k8=np.zeros((BH, N, d), np.int8),
               v8=np.zeros((BH, N, d), np.int8),
               sq=np.zeros((BH, T), np.float32), sk=np.zeros((BH, T), np.float32),
               sv=np.zeros((BH, T), np.float32))
    if tiles:
        out.update(p8=np.zeros((BH, N, N), np.uint8), sp=np.zeros((BH, N, T)))
    rc = _load().oracle_fwd_sel(BH, N, d, blk, flags, _default_tau(d, tau), _p(q), _p(k), _p(v), _p(qsel),
                            _p(out["o"]), _p(out["lse"]), _p(out["mu_k"]), _p(out["mu_q"]),
                            _p(out["bias"]), _p(out["q8"]), _p(out["k8"]), _p(out["v8"]),
                            _p(out["sq"]), _p(out["sk"]), _p(out["sv"]), _p(out.get("p8")), _p(out.get("sp")))
    if rc:
        raise ValueError("oracle_fwd: bad shape")
    return out


def bwd(q, k, v, o_stored, do, lse, *, causal=False, k_smooth=True, q_smooth=False, quant=True,
        blk=128, tau=None, tiles=False, p_u8=False, p_col=False, ds_fine=False, q_blocks=None, k_blocks=None):
    """Alg. 2 per head.  o_stored is the O the forward stored (A15).

    tiles=True also returns the per-tile quantised P^ / dS^ ([BH, N q, N kv] uint8 / int8, tile (i, j) at
    rows i*blk.., columns j*blk..), their psi scales s_P / s_dS ([BH, T i, T j] fp32) and the
    pre-psi dS ([BH, N, N] double); tiles a causal run skips stay zero.  p_col=True: psi(P) per key
    column of each tile (ORC_P_COL); the dumped s_P is then the tile's largest column scale.
    ds_fine=True: psi(dS) per query row for dQ and per key column for dK (ORC_DS_FINE); the dumped dS^
    is then the dK operand.
    q_blocks / k_blocks (either given): process only the tiles of these query / key blocks; dQ is
    computed for q_blocks and dK, dV for k_blocks (other rows stay zero), bitwise as in the full run."""
    q, k, v, o_stored, do, lse = map(_f64, (q, k, v, o_stored, do, lse))
    BH, N, d = q.shape
    T = -(-N // blk)  # ceil: a ragged N has a short last block (reading A33)
    if q_blocks is not None or k_blocks is not None:
        qsel, ksel = _sel(q_blocks or [], BH, T), _sel(k_blocks or [], BH, T)
    else:
        qsel = ksel = None
    flags = _flags(causal, k_smooth, q_smooth, quant, p_u8, p_col, ds_fine)
    out = dict(dq=np.zeros((BH, N, d)), dk=np.zeros((BH, N, d)), dv=np.zeros((BH, N, d)),
               delta=np.zeros((BH, N)), do8=np.zeros((BH, N, d), np.int8),
               sdo=np.zeros((BH, T), np.float32))
    if tiles:
        out.update(p8=np.zeros((BH, N, N), np.uint8), sp=np.zeros((BH, T, T), np.float32),
                   ds8=np.zeros((BH, N, N), np.int8), sds=np.zeros((BH, T, T), np.float32),
                   ds=np.zeros((BH, N, N)))
    rc = _load().oracle_bwd_sel(BH, N, d, blk, flags, _default_tau(d, tau), _p(q), _p(k), _p(v),
                            _p(o_stored), _p(do), _p(lse), _p(qsel), _p(ksel), _p(out["dq"]), _p(out["dk"]),
                            _p(out["dv"]), _p(out["delta"]), _p(out["do8"]), _p(out["sdo"]),
                            _p(out.get("p8")), _p(out.get("sp")), _p(out.get("ds8")), _p(out.get("sds")),
                            _p(out.get("ds")))
    if rc:
        raise ValueError("oracle_bwd: bad shape")
    return out


def fpa(q, k, v, do=None, *, causal=False, tau=None, intermediates=False):
    """Full-precision attention fwd (+bwd if do given), materialising N x N."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    BH, N, d = q.shape
    do = None if do is None else _f64(do)
    out = dict(o=np.zeros((BH, N, d)), lse=np.zeros((BH, N)))
    if do is not None:
        out.update(dq=np.zeros((BH, N, d)), dk=np.zeros((BH, N, d)), dv=np.zeros((BH, N, d)))
    if intermediates:
        out.update(P=np.zeros((BH, N, N)))
        if do is not None:
            out.update(dP=np.zeros((BH, N, N)), dS=np.zeros((BH, N, N)), delta=np.zeros((BH, N)))
    rc = _load().oracle_fpa(BH, N, d, CAUSAL if causal else 0, _default_tau(d, tau),
                            _p(q), _p(k), _p(v), _p(do), _p(out["o"]), _p(out["lse"]),
                            _p(out.get("dq")), _p(out.get("dk")), _p(out.get("dv")),
                            _p(out.get("P")), _p(out.get("dP")), _p(out.get("dS")),
                            _p(out.get("delta")))
    if rc:
        raise ValueError("oracle_fpa: bad shape")
    return out
