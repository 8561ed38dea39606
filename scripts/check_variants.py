"""Quick correctness probe of library builds (SAGE_LIB variants): one small fwd+bwd per head dim vs the oracle.
  SAGE_LIB=... CUDA_LAUNCH_BLOCKING=1 python scripts/check_variants.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2603_02170_b200 import sage  # noqa: E402
from paper_2603_02170_b200.inputs import make_inputs  # noqa: E402

for d, causal, qs, f8 in ((64, True, False, False), (128, True, False, False), (128, False, True, False),
                         (64, True, False, True), (128, False, False, True)):
    B, H, N = 1, 2, 384
    q, k, v, do = make_inputs(B, H, N, d, "outlier_kq", seed=5 + d)
    qd, kd, vd, dod = (t.cuda() for t in (q, k, v, do))
    try:
        o, lse, ctx = sage.forward(qd, kd, vd, causal=causal, q_smooth=qs, pv_fp8=f8)
        dq, dk, dv = sage.backward(ctx, vd, o, lse, dod)
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print(os.environ.get("SAGE_LIB"), d, causal, qs, "FAILED", str(e)[:200])
        sys.exit(1)
    f64 = lambda t: t.float().cpu().numpy().astype(np.float64).reshape(B * H, N, d)
    f = oracle.fwd(f64(q), f64(k), f64(v), causal=causal, q_smooth=qs, pv_fp8=f8)
    bf = lambda x: torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    b = oracle.bwd(f64(q), f64(k), f64(v), bf(f["o"]), f64(do), f["lse"], causal=causal, q_smooth=qs)
    rel = {n: float(np.linalg.norm(bf(r) - f64(g)) / np.linalg.norm(bf(r))) for n, r, g in
           (("o", f["o"], o), ("dq", b["dq"], dq), ("dk", b["dk"], dk), ("dv", b["dv"], dv))}
    print(os.environ.get("SAGE_LIB", "prod").split("/")[-1], d, causal, qs, "fp8" if f8 else "", {n: f"{x:.2e}" for n, x in rel.items()})
