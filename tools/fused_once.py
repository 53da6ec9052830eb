"""One C2 solve with coarse fusion (for ncu): python tools/fused_once.py FUSE_POINTS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2307_00124_b200 as B  # noqa: E402

kw = dict(bench.SOLVES["C2_2d_vcycles"])
kw["cycles"] = 2
mg = B.Multigrid(B.mg_config(**kw, fuse_points=int(sys.argv[1])))
mg.solve()
B.device_sync()
print("ok")
