"""FMG time to discretisation accuracy, second sweep: coarse-solve sweeps and the coarsest
level for the cheap V-cycles.  python tools/fmg_sweep2.py"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402
from bench import sine_accuracy  # noqa: E402

d, l, p = 3, 9, 24
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)
for (nu1, nu2), cyc, nc, lc in itertools.product(((1, 1), (2, 0), (2, 1), (1, 2)), (2,),
                                                 (16, 32, 64), (2, 3)):
    kw = dict(d=d, l_fine=l, l_coarse=lc, cycles=cyc, rhs_kind=1, fmg=True, p=p, nu1=nu1, nu2=nu2,
              n_coarse=nc)
    mg = B.Multigrid(B.mg_config(**kw))
    mg.solve(use_graph=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mg.solve(use_graph=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
    acc = sine_accuracy(d, l, x, e)
    print(f"V({nu1},{nu2}) n_ir={cyc} n_coarse={nc:2d} l_coarse={lc}  {sorted(ts)[1]:7.2f} ms  "
          f"alg/disc={acc['alg_over_disc']:7.3f}  ops={len(tr)}", flush=True)
    del mg
