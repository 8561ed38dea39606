"""K4 pipeline timeline (profiling only): run the C-config bwd with SAGE_ABLATE|8 and print
clock64 event stamps per tile for one CTA (cycles relative to its first event).

  SAGE_ABLATE=8 python scripts/trace_bwd.py [C2] [cta]
"""
import ctypes, os, sys
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("SAGE_LIB", os.path.join(_ROOT, "paper_2603_02170_b200", "libsage_trace.so"))
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_02170_b200 import sage
from paper_2603_02170_b200.inputs import CONFIGS, config_inputs

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c = CONFIGS[cfg]
q, k, v, do = (t.cuda() for t in config_inputs(c))
kw = dict(causal=c.causal, k_smooth=c.k_smooth, q_smooth=c.q_smooth)
for _ in range(3):
    o, lse, ctx = sage.forward(q, k, v, **kw)
    sage.backward(ctx, v, o, lse, do)
torch.cuda.synchronize()
buf = np.zeros(2 * 4 * 64 * 24, dtype=np.uint64)
sage.lib().sage_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), buf.nbytes)
which = 1 if os.environ.get('TRACE_FWD') else 0
tr = buf.reshape(2, 4, 64, 24)[which][cta].astype(np.int64)
names = ["S_iss", "dV_iss", "dP_iss", "dKQ_iss", "-", "c_sfull", "c_pready", "c_dpfull", "c_dsready", "c_dstfree",
         "d_dvfull", "d_dkfull", "d_dqfull", "d_dqdone", "tma_st", "c_ptfree",
         "c_ld0", "m_pready", "c_ldall", "c_tmax", "m_dsrdy", "c_bar1", "m_qfull", "c_st3"]
if which:
    names = ["S_iss", "PV_iss", "c_sfull", "c_pass1", "c_pfull", "-", "m_pfull"] + ["-"] * 17
base = tr[tr > 0].min()
rows = [t for t in range(64) if tr[t].any()]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for t in rows:
    print(f"{t:4d} " + " ".join(f"{(x - base) if x else -1:8d}" for x in tr[t]))
if len(rows) > 4:
    a, b = rows[2], rows[-2]
    col = names.index("S_iss")
    print("per-tile period (S_iss):", (tr[b][col] - tr[a][col]) / (b - a))
