"""Run one sharded solve (in-process group) against the unsharded one; for debugging.
usage: python tools/shard_debug.py d l world min_planes [fmg]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402

d, l, world, minp = (int(a) for a in sys.argv[1:5])
fmg = len(sys.argv) > 5 and sys.argv[5] == "fmg"
cfg = B.mg_config(d=d, l_fine=l, cycles=1 if fmg else 2, rhs_kind=1, fmg=fmg, p=20)
ref = B.Multigrid(cfg)
ref.solve()
xr, qr, er, hr, tr = ref.result()
mg = B.Multigrid(cfg, world=world, min_planes=minp)
try:
    mg.solve()
    B.device_sync()
except Exception as ex:  # noqa: BLE001
    print("solve failed:", ex)
    try:
        B.device_sync()
    except Exception as ex2:  # noqa: BLE001
        print("sync:", ex2)
    raise
x, q, e, h, t = mg.result()
parts = []
for i in range(mg.local):
    xv, rv, rk, ls = mg.rank_result(i)
    parts.append(xv.download()[0])
xs = np.concatenate(parts)
print("ls", ls, "e", e, er, "x equal", np.array_equal(xs, xr), "hist", h == hr)
for i, (a, b) in enumerate(zip(t, tr)):
    if a != b:
        print("first trace diff at", i, a, b)
        break
