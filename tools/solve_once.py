"""Run one solve of a BASELINE config (for ncu launch lists): python tools/solve_once.py C2"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00124_b200 as B
import bench

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
kw = dict(next(v for k, v in bench.SOLVES.items() if k.startswith(name)))
p = kw.pop("p")
mg = B.Multigrid(B.mg_config(**kw, p=p))
mg.solve(use_graph=False)
B.device_sync()
x, q, e, hist, tr = mg.result()
print(name, "ops", len(tr), "final residual", hist[-1])
