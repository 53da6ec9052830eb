import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ob
import ctypes as C, numpy as np, sys
d,l,p,cyc=map(int,sys.argv[1:5])
cfg=ob.mg_config(d,l,cycles=cyc,x0_random=True,rhs_kind=int(os.environ.get("RHS", "2")), p=p)
L=ob.lib(); n=((1<<l)-1)**d
x=ob.OBlock(np.zeros(n,np.int64),1,0); hist=np.zeros(4096); tr=(ob.TraceRec*200000)()
res=ob.MgResult(); res.x=x.c(); res.res_history=hist.ctypes.data_as(C.POINTER(C.c_double)); res.trace=tr; res.trace_cap=200000
st=L.ob_mg_run(C.byref(cfg),C.byref(res)); print("st",st,res.n_trace,res.n_history, hist[:res.n_history])
for t in tr[max(0,res.n_trace-6):res.n_trace]: print(t.step,t.level,t.w_out,t.w_tmp,t.gm,t.ge,t.overflow,t.underflow,t.recomputed)
