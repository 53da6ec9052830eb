import sys
sys.path.insert(0, '.')
import paper_2307_00124_b200 as B
L = int(sys.argv[1]); fmg = sys.argv[2] == '1'
cfg = B.mg_config_ref(L, 1.6, 0.3, w=20, wdot=16, wcheck=24, cycles=1, fmg=fmg, rhs_kind=1, d=2)
mg = B.Multigrid(cfg)
mg.solve(use_graph=False)
x, q, e, hist, tr = mg.result(trace_cap=1 << 14)
print("ok", L, fmg, hist)
