"""Extra residual probes (python tools/probe_extra.py [ops]): 1-D residual at config-1 size
and at a large n (the %HBM claim for 1-D needs n beyond L2), and with
`ops` every fine-level op of config 5 (3-D 1023^3, int64 p = 48)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
for l in (20, 26, 28):
    r = bench.measure_residual(B, torch, stream, 1, l, 16, 4, steps=50 if l < 26 else 10)
    print(f"1-D l={l}", json.dumps(r), flush=True)
if "ops" in sys.argv[1:]:
    torch.cuda.empty_cache()
    print(json.dumps(bench.measure_ops(B, torch, stream, 3, 10, 48, steps=5, s=8)), flush=True)
