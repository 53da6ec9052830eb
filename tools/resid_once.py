"""Run one config's fine-level residual a few times (for ncu captures).

usage: python tools/resid_once.py d l p mant_bytes [steps] [bulk=1]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00124_b200 as B  # noqa: E402

d, l, p, mb = (int(a) for a in sys.argv[1:5])
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
B.set_kernel_path(bulk=(sys.argv[6] != "0") if len(sys.argv) > 6 else True)
x = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 1, 1)
b = (B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 1, 2) if d == 1 else
     B.gen_sine(B.BfpVec.grid(d, l, mb), p))  # config 1: uniform rhs
r = B.BfpVec.grid(d, l, mb)
B.residual(x, b, p, p + 5, B.Scalar(1 << 14, 16, 2 * l + 8), out=r)
g = B.inf_norm_upper(r).c()
L = B.lib()
for _ in range(steps):
    assert L.bfp_stencil_gemv(x.h, b.h, B.bfp_minus_one().c(), B.bfp_one().c(), 0, p, p + 5, g, 0,
                              r.h, None) == 0
B.device_sync()
print("ok", r.header().flags)
