"""A/B: fine-level op throughput with the library named by $BFPMG_LIB.
python tools/ab_ops.py d l op[,op...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

d, l = int(sys.argv[1]), int(sys.argv[2])
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
for op in sys.argv[3].split(","):
    r = bench.measure_ops(B, torch, stream, d, l, 24 if d == 3 else 20, steps=20, only=op)
    o = r["ops"][op]
    print(f"{os.environ.get('BFPMG_LIB', 'default')[-30:]:30s} d={d} l={l} {op:16s} "
          f"{o['kernel_ms'] * 1e3:8.1f} us  {o['hbm_frac']:.3f}", flush=True)
