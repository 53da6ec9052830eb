"""Per-op kernel time and HBM fraction over the upper levels of a hierarchy (the sizes a
solve spends its bandwidth on): python tools/ops_levels.py d p l_max l_min"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

d, p, lmax, lmin = (int(a) for a in sys.argv[1:5])
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
peak = bench.hbm_peak()[0] if hasattr(bench, "hbm_peak") else 6465.5
for l in range(lmax, lmin - 1, -1):
    r = bench.measure_ops(B, torch, stream, d, l, p, steps=30)["ops"]
    n = (2 ** l) ** d
    print(f"l={l}: " + "  ".join(
        f"{k[:8]} {v['kernel_ms'] * 1e3:6.1f}us {v['hbm_frac']:.2f} (+{v['kernel_ms'] * 1e3 * (1 - v['hbm_frac']):.1f})"
        for k, v in r.items()))
