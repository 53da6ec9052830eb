"""First trace record that differs between per-op launches and the fused coarse engine.
python tools/fuse_debug.py c1|c4 [fuse_points]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

CASES = {
    "c1": (dict(d=1, l_fine=14, cycles=10, x0_random=True, rhs_kind=0, pd=[28] * 32, w_add_cap=4), 16),
    "c1s": (dict(d=1, l_fine=6, cycles=2, x0_random=True, rhs_kind=0, pd=[28] * 32, w_add_cap=4), 16),
    "c4": (dict(d=3, l_fine=4, cycles=2, rhs_kind=1, fmg=True, nu2=1), 24),
    "c4s": (dict(d=3, l_fine=2, cycles=2, rhs_kind=1, fmg=True, nu2=1), 24),
}
name = sys.argv[1]
fp = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
kw, p = CASES[name]
res = []
for f in (0, fp):
    mg = B.Multigrid(B.mg_config(**kw, p=p, fuse_points=f))
    mg.solve(use_graph=False)
    res.append(mg.result(trace_cap=1 << 16))
(x0, q0, e0, h0, t0), (x1, q1, e1, h1, t1) = res
print("x equal", np.array_equal(x0, x1), "e", e0, e1, "q", q0, q1, "hist equal", h0 == h1)
print("hist", h0[:6], h1[:6])
n = 0
for i, (a, b) in enumerate(zip(t0, t1)):
    if tuple(a) != tuple(b):
        print("trace", i, B.STEP_NAMES[a[0]], "level", a[1], "ref", tuple(a), "fused", tuple(b))
        n += 1
        if n > 6:
            break
print("trace records", len(t0), len(t1), "mismatches shown", n)

if os.environ.get("BFPMG_LIB"):
    import ctypes as C
    ops = (C.c_int * (4 * 64))()
    B.lib().bfp_dbg_coarse_ops(ops, 64)
    kn = ["gemv", "jacobi", "scal", "axpby", "restrict", "prolong", "pcorr", "zero"]
    sn = ["none", "fastq", "fastn", "generic", "zero"]
    for i in range(40):
        k, a, b, c = ops[4 * i:4 * i + 4]
        print(f"   {i:3d} {kn[(k >> 4) & 7]:9s} {sn[k & 15] if (k & 15) < 5 else k & 15:8} e={a:6d} mx={b:12d} mn={c:12d}")
