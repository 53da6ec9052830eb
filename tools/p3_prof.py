"""Per-phase clocks of the 3-D prolongation march (block 0, thread 0), -DBFP_P3_TIMING build:
BFPMG_LIB=paper_2307_00124_b200/_ab/p3t/libbfpmg_b200.so python tools/p3_prof.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
out = (C.c_longlong * 8)()
for op in ("prolong", "prolong_correct"):
    B.lib().bfp_dbg_p3(out)
    r = bench.measure_ops(B, torch, stream, 3, 9, 24, steps=5, only=op, s=4)["ops"][op]
    B.lib().bfp_dbg_p3(out)
    v = list(out)
    n = max(v[4], 1)
    print(op, "hbm_frac %.3f" % r["hbm_frac"], "steps", v[4],
          "per step: wait %.0f compute+store %.0f syncthreads %.0f issue %.0f clk" %
          (v[0] / n, v[1] / n, v[2] / n, v[3] / n))
