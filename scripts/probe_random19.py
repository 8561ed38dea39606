import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, oracle
from paper_2603_02170_b200 import sage
from paper_2603_02170_b200.inputs import make_inputs
from tests.metrics import f64, round_bf16, rel_l2
B,H,N,d=2,1,1024,64
q,k,v,do=make_inputs(B,H,N,d,"outlier_kq",seed=3019)
for var in ("none","p_u8"):
  for ks in (False, True):
    kw={} if var=="none" else {var:True}
    qd,kd,vd,dod=(t.cuda() for t in (q,k,v,do))
    o,lse,ctx=sage.forward(qd,kd,vd,causal=True,k_smooth=ks,**kw)
    dq,dk,dv=sage.backward(ctx,vd,o,lse,dod); torch.cuda.synchronize()
    sel=lambda t: f64(t).reshape(B*H,N,d)
    f=oracle.fwd(sel(q),sel(k),sel(v),causal=True,k_smooth=ks,p_u8=var=="p_u8")
    b=oracle.bwd(sel(q),sel(k),sel(v),round_bf16(f["o"]),sel(do),f["lse"],causal=True,k_smooth=ks,p_u8=var=="p_u8")
    fp=oracle.fpa(sel(q),sel(k),sel(v),sel(do),causal=True)
    print(var, "ks", ks, "gpu-vs-QO dq %.2e dk %.2e | QO-vs-FPA dq %.3f | GPU-vs-FPA dq %.3f" % (rel_l2(round_bf16(b["dq"]),sel(dq)), rel_l2(round_bf16(b["dk"]),sel(dk)), rel_l2(fp["dq"], b["dq"]), rel_l2(fp["dq"], sel(dq))))
