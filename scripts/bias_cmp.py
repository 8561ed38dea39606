"""Dump the Q-smoothing bias of one small C3-like forward (SAGE_LIB selects the build) to an .npy file, or
compare two dumps bitwise: python scripts/bias_cmp.py out.npy | python scripts/bias_cmp.py a.npy b.npy"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

if len(sys.argv) == 3:
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    print("bias bitwise equal:", a.shape, bool((a.view(np.uint32) == b.view(np.uint32)).all()))
    sys.exit(0)
import torch  # noqa: E402
from paper_2603_02170_b200 import sage  # noqa: E402
from paper_2603_02170_b200.inputs import make_inputs  # noqa: E402

outs = []
for N, d in ((4096, 128), (1000, 64), (300, 128)):
    q, k, v, _ = make_inputs(1, 4, N, d, "outlier_kq", seed=77 + N)
    o, lse, ctx = sage.forward(q.cuda(), k.cuda(), v.cuda(), causal=True, q_smooth=True)
    torch.cuda.synchronize()
    outs.append(ctx.view()["bias"].cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(outs))
