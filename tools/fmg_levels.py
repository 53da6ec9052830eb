"""FMG error vs the discrete solution as a function of the finest level (the
progressive schedule p_l = 4 + 2(l-3) is level-local, so each run extends the last)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2307_00124_b200 as B  # noqa: E402
from bench import sine_accuracy  # noqa: E402

prog = [0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]
variants = {
    "prog": dict(p=prog),
    "prog_nc64": dict(p=prog, n_coarse=64),
    "prog_c2": dict(p=prog, cycles=2),
    "prog_c3": dict(p=prog, cycles=3),
    "prog_pc+4": dict(p=prog, pc=[v + 4 if v else 0 for v in prog]),
    "prog+4": dict(p=[v + 4 if v else 0 for v in prog]),
}
for name, extra in variants.items():
    row = []
    for lf in range(5, 14):
        kw = dict(d=2, l_fine=lf, l_coarse=3, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True)
        kw.update(extra)
        mg = B.Multigrid(B.mg_config(**kw))
        mg.solve()
        x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
        a = sine_accuracy(2, lf, x, e)
        row.append(f"{a['err_vs_discrete']:.1e}/{a['alg_over_disc']:.0f}")
    print(f"{name:10s}", " ".join(row), flush=True)
