"""One fwd+bwd per variant at small shapes, for compute-sanitizer (racecheck / synccheck / memcheck).

  compute-sanitizer --tool racecheck python scripts/sanitize_run.py
Shapes: C1 (N=128) and N=384 / 256 (multi-tile), d = 64 and 128, causal and not, every K2/K4 variant the
library instantiates (default, Q-smoothing, P_U8, P_COLSCALE, FINE_BWD, DETERMINISTIC, FP32_OUT; fp16 I/O
on the default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2603_02170_b200 import sage  # noqa: E402
from paper_2603_02170_b200.inputs import make_inputs  # noqa: E402

VARIANTS = [dict(), dict(q_smooth=True), dict(p_u8=True), dict(p_colscale=True), dict(fine_bwd=True),
            dict(deterministic=True), dict(fp32_out=True)]
only = os.environ.get("SAN_ONLY")
n = 0
for N, d, causal in ((128, 64, True), (384, 64, False), (384, 128, True), (256, 128, False)):
    for vi, var in enumerate(VARIANTS):
        if only and str(vi) not in only.split(","):
            continue
        for dtype in ((torch.bfloat16, torch.float16) if vi == 0 else (torch.bfloat16,)):
            q, k, v, do = (t.cuda() for t in make_inputs(1, 2, N, d, "outlier_kq", seed=N + d, dtype=dtype))
            o, lse, ctx = sage.forward(q, k, v, causal=causal, **var)
            sage.backward(ctx, v, o, lse, do)
            torch.cuda.synchronize()
            n += 1
print(f"sanitize_run: {n} fwd+bwd runs completed")
