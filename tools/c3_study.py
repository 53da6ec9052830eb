"""Config 3 (2-D FMG, progressive precision p_l = 4 + 2 (l - 3)): qcomp vs nnqcomp vs hybrid on
the same schedule, and schedule variants, with the max-norm and energy-norm errors against
the discrete solution.  python tools/c3_study.py [l_fine]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2307_00124_b200 as B  # noqa: E402
from bench import sine_accuracy  # noqa: E402

lf = int(sys.argv[1]) if len(sys.argv) > 1 else 13
stream = torch.cuda.current_stream()
B.set_stream(stream.cuda_stream)


def energy(d, l, m, e):
    """Energy-norm error |u - u_h|_A / |u_h|_A against the discrete solution of the sine rhs."""
    n = (1 << l) - 1
    h = 2.0 ** -l
    s = np.sin(np.pi * h * np.arange(1, n + 1))
    lam = 4 * d / h ** 2 * np.sin(np.pi * h / 2) ** 2
    uh = (d * np.pi ** 2 / lam) * np.multiply.outer(s, s)
    u = np.ldexp(m.astype(np.float64), e).reshape(n, n)
    err = u - uh

    def anorm(v):
        p = np.pad(v, 1)
        av = (4 * p[1:-1, 1:-1] - p[:-2, 1:-1] - p[2:, 1:-1] - p[1:-1, :-2] - p[1:-1, 2:]) / h ** 2
        return float(np.sqrt(abs((v * av).sum()) * h * h))
    return anorm(err) / anorm(uh), anorm(err)


def sched(base, step, l0=3):
    return [0, 0, 0] + [base + step * (l - l0) for l in range(l0, 32)][:29]


variants = {
    "frozen p=4+2(l-3)": dict(p=sched(4, 2)),
    "p=4+2(l-3), wdot=p+4": dict(p=sched(4, 2), pd=sched(8, 2)),
    "p=4+2(l-3), wdot=p+4, wcheck=p+8": dict(p=sched(4, 2), pd=sched(8, 2), pc=sched(12, 2)),
    "p=8+2(l-3)": dict(p=sched(8, 2)),
    "p=6+2(l-3), wdot=p+2": dict(p=sched(6, 2), pd=sched(8, 2)),
}
for name, kw in variants.items():
    for mode, nn in (("qcomp", False), ("nnqcomp", True), ("hybrid", "hybrid")):
        for cyc in (1, 2):
            cfg = B.mg_config(d=2, l_fine=lf, l_coarse=3, cycles=cyc, rhs_kind=1, fmg=True,
                              nonnormalized=nn, **kw)
            mg = B.Multigrid(cfg)
            mg.solve(use_graph=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mg.solve(use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
            acc = sine_accuracy(2, lf, x, e)
            en_rel, en_abs = energy(2, lf, x, e)
            rc = sum(1 for t in tr if t[8])
            print(f"{name:36s} {mode:8s} n_ir={cyc} {e0.elapsed_time(e1):6.2f} ms  "
                  f"max-norm alg/disc={acc['alg_over_disc']:10.3g}  energy rel={en_rel:9.3g}  "
                  f"res {hist[0]:.3g}->{hist[-1]:.3g}  recomputes={rc}", flush=True)
            del mg
