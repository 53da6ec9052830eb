"""int64 Jacobi (3-D, l=10) at p=32 and p=48: fraction of the HBM peak (A/B with BFPMG_LIB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
for p in (32, 40, 48):
    best = 0
    for rep in range(3):
        r = bench.measure_ops(B, torch, stream, 3, 10, p, steps=6, only="jacobi", s=8)["ops"]["jacobi"]
        best = max(best, r["hbm_frac"])
    print(f"p={p} jacobi {best:.3f}")
