"""Run one fine-level op a few times (for ncu): python tools/op_once.py d l op [steps] [p] [s]
op in residual, jacobi, scal, axpby, restrict, prolong, prolong_correct"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

d, l, op = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
p = int(sys.argv[5]) if len(sys.argv) > 5 else (24 if d == 3 else 20)
s = int(sys.argv[6]) if len(sys.argv) > 6 else 4
r = bench.measure_ops(B, torch, stream, d, l, p, steps=steps, only=op, s=s)
print(r)
