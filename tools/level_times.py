"""Solve time vs finest level (graph replay, CUDA events): T(l) - T(l-1) is the cost of
level l inside the solve, T(l_small) the latency floor of the coarse hierarchy.
python tools/level_times.py C4_3d_fmg_n2 [l_min]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4_3d_fmg_n2"
base = dict(bench.SOLVES[name])
lmin = int(sys.argv[2]) if len(sys.argv) > 2 else 2
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
B.set_stream(stream.cuda_stream)
prev = 0.0
for l in range(lmin, base["l_fine"] + 1):
    kw = dict(base, l_fine=l)
    p = kw.pop("p")
    if "l_coarse" in kw and kw["l_coarse"] > l:
        continue
    mg = B.Multigrid(B.mg_config(**kw, p=p))
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
    t = sorted(ts)[len(ts) // 2]
    _, _, _, hist, tr = mg.result()
    print(f"{name} l_fine={l:2d} ms={t:8.3f}  delta={t - prev:8.3f}  ops={len(tr)}", flush=True)
    prev = t
    del mg
