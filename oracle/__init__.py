"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for SageBwd (arXiv 2603.02170).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2603_02170_b200``) never imports, links or calls it.

Parity status per function:
  * ``psi_block``, ``psi_token_row``            pinned (SPEC worked examples, half-step bound)
  * ``fwd`` / ``bwd`` with ``quant=False``       pinned (== FPA <= 1e-9; FPA pinned by finite differences)
  * ``fwd`` / ``bwd`` with ``quant=True``        pinned (Table 1 trend/values, smoothing identities, grid fixed points)
  * ``fpa``                                     pinned (finite differences, closed forms, App. B bound)
  * ``qknorm.forward`` / ``qknorm.backward``    pinned (closed forms, unit RMS, finite differences)
  * ``e4m3``, ``psi_block_e4m3``, ``fwd(pv_fp8)`` pinned (torch float8_e4m3fn, exact-P limit, FPA closeness)
  * ``policy.attention`` (per-MatMul precision)  pinned (exact policy == fpa, per-site dependency pattern,
                                                 SageBwd policy tracks the tiled quantised oracle)
"""
from . import policy, qknorm
from .oracle import (CAUSAL, K_SMOOTH, Q_SMOOTH, QUANT_OFF, build, fpa, fwd, bwd, e4m3,
                     psi_block, psi_block_e4m3, psi_token_row, set_threads, max_threads)

__all__ = ["policy", "qknorm", "CAUSAL", "K_SMOOTH", "Q_SMOOTH", "QUANT_OFF", "build", "fpa", "fwd", "bwd",
           "psi_block", "psi_token_row", "set_threads", "max_threads", "e4m3", "psi_block_e4m3"]
