"""int64-storage fine-level ops (BASELINE config 5 widths): residual / Jacobi kernel time
and fraction of the HBM peak.  python tools/ab_c5.py [l] [p,p,...] [op,op,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

l = int(sys.argv[1]) if len(sys.argv) > 1 else 10
ps = [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "32,48").split(",")]
ops = (sys.argv[3] if len(sys.argv) > 3 else "residual,jacobi").split(",")
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
tag = os.environ.get("BFPMG_LIB", "default")[-30:]
for p in ps:
    for op in ops:
        r = bench.measure_ops(B, torch, stream, 3, l, p, steps=10, only=op, s=8)
        o = r["ops"][op]
        print(f"{tag:30s} l={l} p={p} {op:10s} {o['kernel_ms'] * 1e3:9.1f} us  {o['hbm_frac']:.3f}",
              flush=True)
        torch.cuda.empty_cache()
