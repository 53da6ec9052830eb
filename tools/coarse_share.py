"""Where a C4 FMG solve spends its time: the whole solve, the FMG of its coarse part alone
(levels <= lc), and V-cycle descents from level lc (what levels lc+1 .. 9 add on the coarse
levels).  python tools/coarse_share.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)


def t(**kw):
    mg = B.Multigrid(B.mg_config(**kw))
    mg.solve(use_graph=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        mg.solve(use_graph=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    n = mg.launches()
    del mg
    return sorted(ts)[2], n


base = dict(d=3, rhs_kind=1, p=24, nu2=0, n_coarse=32, l_coarse=3)
full, nl = t(l_fine=9, cycles=2, fmg=True, **base)
print(f"FMG(9) V(2,0)x2: {full:.2f} ms, {nl} launches")
for lc in (4, 5, 6, 7, 8):
    f, n1 = t(l_fine=lc, cycles=2, fmg=True, **base)
    v, n2 = t(l_fine=lc, cycles=2, fmg=False, **base)  # 2 IR-V cycles at level lc
    desc = 9 - lc  # FMG levels above lc, each adding one 2-cycle IR through level lc
    print(f"lc={lc}: FMG({lc}) {f:.3f} ms ({n1} launches), 2 x IR-V({lc}) {v:.3f} ms ({n2}); "
          f"levels <= {lc} inside FMG(9) ~ {f + desc * v:.2f} ms")
