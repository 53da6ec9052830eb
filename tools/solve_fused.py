import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00124_b200 as B
mg = B.Multigrid(B.mg_config(2, 12, cycles=2, rhs_kind=1, p=20, fuse_points=int(os.environ.get("FUSE", "256"))))
mg.solve()
B.device_sync()
print("ok")
