"""Fine-level ops of C2, C4, C5 (fractions of the HBM peak), best of two passes:
python tools/ops_now.py [op ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
only = sys.argv[1:] or None
res = {}
for rep in range(2):
    for cfg, (d, l, p, s, steps) in {"C2": (2, 12, 20, 4, 20), "C4": (3, 9, 24, 4, 20),
                                     "C5": (3, 10, 48, 8, 4)}.items():
        for op in (only or ["residual", "jacobi", "scal", "axpby", "restrict", "prolong",
                            "prolong_correct"]):
            r = bench.measure_ops(B, torch, stream, d, l, p, steps=steps, only=op, s=s)["ops"][op]
            k = (cfg, op)
            res[k] = max(res.get(k, 0), r["hbm_frac"])
for (cfg, op), v in res.items():
    print(f"{cfg:3s} {op:16s} {v:.3f}")
