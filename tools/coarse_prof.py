"""Per-phase clock totals of the coarse engine (a -DBFP_COARSE_TIMING build, tools/ab_build.sh):
BFPMG_LIB=paper_2307_00124_b200/_ab/ctime/libbfpmg_b200.so python tools/coarse_prof.py C2 4096"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

name, fp = sys.argv[1], int(sys.argv[2])
kw = dict(next(v for k, v in bench.SOLVES.items() if k.startswith(name)))
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)
mg = B.Multigrid(B.mg_config(**kw, fuse_points=fp))
mg.solve(use_graph=True)
torch.cuda.synchronize()
out = (C.c_longlong * 16)()
B.lib().bfp_dbg_coarse(out)
mg.solve(use_graph=True)
torch.cuda.synchronize()
B.lib().bfp_dbg_coarse(out)
names = ["griddep_wait", "arena_load", "setup (C->A)", "barrier A", "body | late gamma", "barrier B",
         "totals+core fin", "writeback", "launches", "ops", "barrier C", "generic ops"]
v = list(out)
ops = max(v[9], 1)
print(f"{name} fuse_points={fp}: launches={v[8]} ops={v[9]}")
for k, nm in enumerate(names):
    if k in (8, 9):
        continue
    per = "launch" if k in (0, 1, 7) else "op"
    den = v[8] if per == "launch" else ops
    print(f"  {nm:18s} {v[k]:12d} clk  {v[k] / max(den, 1):9.1f} clk/{per}")

ops = (C.c_int * (4 * 64))()
B.lib().bfp_dbg_coarse_ops(ops, 64)
kn = ["gemv", "jacobi", "scal", "axpby", "restrict", "prolong", "pcorr", "zero"]
print("  last launch, first ops: t32 fetch | post-setup | t32 A->B | totals+core (clk)")
for i in range(40):
    k, a, b, c = ops[4 * i:4 * i + 4]
    print(f"   {i:3d} {k:7d} {a:7d} {b:7d} {c:7d}")
