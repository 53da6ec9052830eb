"""FMG accuracy vs the discrete solution for variants of the C3 / C4 configs.
usage: python tools/accuracy_sweep.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00124_b200 as B  # noqa: E402
from bench import sine_accuracy  # noqa: E402

prog = [0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]
runs = [
    ("C3_l13_nnq_nc16", dict(d=2, l_fine=13, l_coarse=3, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True, p=prog)),
    ("C3_l13_nnq_nc32", dict(d=2, l_fine=13, l_coarse=3, n_coarse=32, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True, p=prog)),
    ("C3_l13_nnq_nc64", dict(d=2, l_fine=13, l_coarse=3, n_coarse=64, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True, p=prog)),
    ("C3_l13_q_nc64", dict(d=2, l_fine=13, l_coarse=3, n_coarse=64, cycles=1, rhs_kind=1, fmg=True, p=prog)),
    ("C3_l13_nnq_nc64_c2", dict(d=2, l_fine=13, l_coarse=3, n_coarse=64, cycles=2, rhs_kind=1, fmg=True, nonnormalized=True, p=prog)),
    ("C4_c1", dict(d=3, l_fine=9, cycles=1, rhs_kind=1, fmg=True, p=24)),
    ("C4_c2", dict(d=3, l_fine=9, cycles=2, rhs_kind=1, fmg=True, p=24)),
    ("C2_fmg_c1", dict(d=2, l_fine=12, cycles=1, rhs_kind=1, fmg=True, p=20)),
    ("C2_fmg_c2", dict(d=2, l_fine=12, cycles=2, rhs_kind=1, fmg=True, p=20)),
]
for name, kw in runs:
    mg = B.Multigrid(B.mg_config(**kw))
    mg.solve(use_graph=True)
    B.device_sync()
    t = time.time()
    mg.solve(use_graph=True)
    B.device_sync()
    ms = (time.time() - t) * 1e3
    x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
    acc = sine_accuracy(kw["d"], kw["l_fine"], x, e)
    print(f"{name:18s} {ms:8.2f} ms  err_h={acc['err_vs_discrete']:.3e} disc={acc['disc_err']:.3e} "
          f"ratio={acc['alg_over_disc']:.2f} res0={hist[0]:.3e} resN={hist[-1]:.3e} "
          f"sat/rc={sum(t_[8] for t_ in tr)}", flush=True)
