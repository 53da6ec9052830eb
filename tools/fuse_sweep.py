"""Solve time vs the coarse-level fusion threshold (fuse_points), results checked equal.
python tools/fuse_sweep.py [C1 C2 ...]   (FUSE_POINTS=0,64,... overrides the thresholds)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
names = sys.argv[1:] or ["C1", "C2", "C4"]
for name in names:
    kw = dict(next(v for k, v in bench.SOLVES.items() if k.startswith(name)))
    ref = None
    for fp in [int(v) for v in os.environ.get("FUSE_POINTS", "0,64,512,4096,32768").split(",")]:
        mg = B.Multigrid(B.mg_config(**kw, fuse_points=fp))
        mg.solve(use_graph=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            mg.solve(use_graph=True)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
        if ref is None:
            ref = (x, e, hist)
        same = np.array_equal(x, ref[0]) and e == ref[1] and hist == ref[2]
        print(f"{name} fuse_points={fp:6d} {ms:8.2f} ms launches={mg.launches():5d} same={same}",
              flush=True)
        del mg
