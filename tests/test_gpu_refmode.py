"""Reference-algorithm parity mode on the GPU vs its big-int
restatement oracle/pyref_refmode.py: Chebyshev V(1,0) cycles, IR and FMG of
P/src/multigrid.cpp:430-518 with the Table-1 gamma chain, 1-D and 2-D p = 1 operators
(2-D: the 9-point bilinear-FEM operator, P = P1 (x) P1, R = P^T), coarsest level 1.
Final iterate, residual history and every trace record must match."""
import pytest

from oracle import pyref as P
from oracle import pyref_refmode as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2307_00124_b200 as B
    B.lib()
    return B


def _levels(v, L):
    return [0] + ([v] * L if isinstance(v, int) else list(v[1:L + 1]))


def _rhs(kind, L, wcheck, seed, fmg, d=1):
    out = {}
    for l in range(1, L + 1):
        if not fmg and l != L:
            continue
        if kind == 1:
            b = P.gen_sine(d, l, wcheck[l])
            if any(b.m):
                b.e -= 2 * l + d
        elif kind == 3:  # the FEM load vector by quadrature, D^-1-scaled
            b = R.fem_rhs(d, l, wcheck[l])
        elif kind == 0:
            b = P.gen_uniform(d, l, wcheck[l], seed, 2)
        else:
            b = P.zero_vec(((1 << l) - 1) ** d, wcheck[l])
        out[l] = b
    return out


CASES = [
    dict(L=6, w=20, wdot=16, wcheck=24, rho=2.02, eta=0.3, cycles=1, fmg=True, rhs=1),
    dict(L=7, w=[0] + [6 + 2 * l for l in range(1, 8)], wdot=[0] + [4 + 2 * l for l in range(1, 8)],
         wcheck=[0] + [10 + 2 * l for l in range(1, 8)], rho=2.02, eta=0.0, cycles=2, fmg=True, rhs=1),
    dict(L=7, w=16, wdot=16, wcheck=20, rho=2.02, eta=0.15, cycles=5, fmg=False, rhs=0, x0=True),
    dict(L=6, w=40, wdot=36, wcheck=44, rho=2.0, eta=0.5, cycles=3, fmg=False, rhs=1),
    dict(L=5, w=12, wdot=12, wcheck=12, rho=2.02, eta=0.3, cycles=2, fmg=False, rhs=2, x0=True),
    # the reference's own right-hand side: FEM load of 9 pi^2 sin(3 pi x) by 2-point Gauss
    dict(L=7, w=20, wdot=16, wcheck=24, rho=2.02, eta=0.3, cycles=1, fmg=True, rhs=3),
    dict(L=6, w=40, wdot=36, wcheck=44, rho=2.0, eta=0.3, cycles=3, fmg=False, rhs=3),
    # the reference's whole setup: rho by power iteration on level min(5, L), FEM load
    dict(L=6, w=24, wdot=20, wcheck=28, rho="auto", eta=0.3, cycles=1, fmg=True, rhs=3),
    # 2-D: rho = lambda_max(D^-1 A) of the 9-point operator is < 2 (Gershgorin); the
    # reference estimates it by power iteration (P/src/linalg.cpp:272-295), injected here
    dict(d=2, L=5, w=20, wdot=16, wcheck=24, rho=1.6, eta=0.3, cycles=1, fmg=True, rhs=1),
    dict(d=2, L=5, w=[0] + [6 + 2 * l for l in range(1, 6)], wdot=[0] + [5 + 2 * l for l in range(1, 6)],
         wcheck=[0] + [10 + 2 * l for l in range(1, 6)], rho=1.6, eta=0.1, cycles=2, fmg=True, rhs=1),
    dict(d=2, L=5, w=16, wdot=16, wcheck=20, rho=1.7, eta=0.2, cycles=4, fmg=False, rhs=0, x0=True),
    dict(d=2, L=6, w=40, wdot=36, wcheck=44, rho=1.6, eta=0.5, cycles=2, fmg=False, rhs=1),
    dict(d=2, L=4, w=8, wdot=8, wcheck=8, rho=1.6, eta=0.3, cycles=2, fmg=False, rhs=2, x0=True),
    dict(d=2, L=5, w=20, wdot=16, wcheck=24, rho=1.6, eta=0.3, cycles=1, fmg=True, rhs=3),
    dict(d=2, L=4, w=40, wdot=36, wcheck=44, rho=1.6, eta=0.3, cycles=2, fmg=False, rhs=3),
    dict(d=2, L=3, w=24, wdot=20, wcheck=28, rho="auto", eta=0.3, cycles=2, fmg=True, rhs=3),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"d{c.get('d', 1)}_L{c['L']}_{'fmg' if c['fmg'] else 'ir'}_w{c['w'] if isinstance(c['w'], int) else 'prog'}_rhs{c['rhs']}{'_rhoauto' if c['rho'] == 'auto' else ''}")
def test_refmode_gpu_vs_pyref(B, case):
    L, d = case["L"], case.get("d", 1)
    w, wd, wc = (_levels(case[k], L) for k in ("w", "wdot", "wcheck"))
    seed = 3
    x0 = P.gen_uniform(d, L, w[L], seed, 1) if case.get("x0") else None
    if case["rho"] == "auto":  # Hierarchy::setup_scaling: oracle restatement vs host code
        from paper_2307_00124_b200 import refmode
        case = dict(case, rho=refmode.estimate_rho(d, min(5, L)))
        assert case["rho"] == R.power_rho(d, min(5, L))
    cfg = R.RefConfig(l_fine=L, w=w, wdot=wd, wcheck=wc, rho=case["rho"], eta=case["eta"],
                      cycles=case["cycles"], fmg=case["fmg"], x0=x0, d=d)
    want = R.RefMg(cfg, _rhs(case["rhs"], L, wc, seed, case["fmg"], d)).run()
    gcfg = B.mg_config_ref(L, case["rho"], case["eta"], w=w, wdot=wd, wcheck=wc,
                           cycles=case["cycles"], fmg=case["fmg"], x0_random=bool(case.get("x0")),
                           rhs_kind=case["rhs"], seed=seed, d=d)
    for graph in (False, True):
        mg = B.Multigrid(gcfg)
        if case["rhs"] == 3:
            from paper_2307_00124_b200 import refmode
            refmode.set_fem_rhs(mg)
        mg.solve(use_graph=graph)
        x, q, e, hist, tr = mg.result(trace_cap=1 << 14)
        assert [tuple(t) for t in tr] == [tuple(t) for t in want.trace], graph
        assert hist == want.history
        assert e == want.x.e and x.tolist() == want.x.m


@pytest.mark.parametrize("d,L", [(1, 4), (2, 3)])
def test_conv_rate_vcycle_columns(B, d, L):
    """conv_rate_vcycle (P/src/multigrid.cpp:572-601): every column (I - B A) e_i of the
    batched GPU run equals the restatement's, and rho_V is a contraction."""
    from paper_2307_00124_b200 import refmode
    w, wd, wc, eta = 20, 16, 24, 0.3
    rho = 2.02 if d == 1 else 1.6
    rate, cols = refmode.conv_rate_vcycle(L, rho, eta, w=w, wdot=wd, wcheck=wc, streams=4, d=d)
    n = ((1 << L) - 1) ** d
    lv = [0] + [w] * L, [0] + [wd] * L, [0] + [wc] * L
    for i in range(n):
        x0 = P.Block([0] * n, wd, 2 - wd)
        x0.m[i] = 1 << (wd - 2)
        cfg = R.RefConfig(l_fine=L, w=lv[0], wdot=lv[1], wcheck=lv[2], rho=rho, eta=eta, cycles=1,
                          fmg=False, x0=x0, d=d)
        want = R.RefMg(cfg, {L: P.zero_vec(n, wc)}).run()
        assert cols[i][1] == want.x.e and cols[i][0].tolist() == want.x.m, i
    assert 0.0 < rate < 1.0


@pytest.mark.parametrize("d,L,w,wd,wc", [(1, 7, 14, 10, 18), (2, 5, 12, 9, 16)])
def test_recompute_table_vs_pyref(B, d, L, w, wd, wc):
    """The reference's Table 2 (cmd_recompute_table, P/src/experiments.cpp:556-600): per
    w_add cap, recomputations and calls at the finest level of the FMG solve
    (SolverTrace::recomputes_at_level / calls_at_level) -- GPU counts equal the
    restatement's, the records' to_line text included, and the counts grow as the cap
    shrinks (the table's own check)."""
    from paper_2307_00124_b200 import refmode
    rho, eta = (2.02, 0.3) if d == 1 else (1.6, 0.3)
    rows = refmode.recompute_table(L, rho, eta, w=w, wdot=wd, wcheck=wc, n_ir=2, d=d)
    lv = [0] + [w] * L, [0] + [wd] * L, [0] + [wc] * L
    prev = -1
    for cap, rec, calls in rows:
        cfg = R.RefConfig(l_fine=L, w=lv[0], wdot=lv[1], wcheck=lv[2], rho=rho, eta=eta, cycles=2,
                          fmg=True, d=d, w_add_cap=cap)
        mg = R.RefMg(cfg, _rhs(1, L, lv[2], 3, True, d))
        mg.run()
        assert (rec, calls) == (mg.recomputes_at_level(L), mg.calls_at_level(L)), cap
        assert rec >= prev, rows
        prev = rec
    assert rows[-1][1] > 0  # cap 0: no headroom, the narrow window recomputes
    # the trace text of one run, line by line (TraceRecord::to_line, :157-163)
    gcfg = B.mg_config_ref(L, rho, eta, w=B.PrecisionSchedule.flat(L, wc, w, wd), cycles=2,
                           fmg=True, rhs_kind=1, d=d, w_add_cap=2)
    mg = B.Multigrid(gcfg)
    mg.solve()
    lines = mg.trace().lines()
    cfg = R.RefConfig(l_fine=L, w=lv[0], wdot=lv[1], wcheck=lv[2], rho=rho, eta=eta, cycles=2,
                      fmg=True, d=d, w_add_cap=2)
    want = R.RefMg(cfg, _rhs(1, L, lv[2], 3, True, d)).run()
    assert len(lines) == len(want.trace)
    for line, t in zip(lines, want.trace):
        assert line == B.TraceRecord(*t).to_line()
        assert line.split()[0] in B.REF_STEP_NAMES


def test_refmode_schedule_validate(B):
    """PrecisionSchedule::validate (P/src/multigrid.cpp:37-44): the reference mode rejects
    schedules that break wcheck >= w >= wdot >= 1, in the mirror and in the C-ABI."""
    s = B.PrecisionSchedule.affine(6, 1, 2, 8, 4, 2)
    s.validate()
    assert s.w[3] == 10 and s.wcheck[3] == 17 and s.wdot[3] == 5
    bad = B.PrecisionSchedule.flat(5, 20, 16, 18)  # wdot > w
    with pytest.raises(ValueError):
        bad.validate()
    with pytest.raises(ValueError):
        B.mg_config_ref(5, 2.02, 0.3, w=bad)
    cfg = B.mg_config_ref(5, 2.02, 0.3, w=16, wdot=18, wcheck=20)  # raw widths: the C-ABI checks
    with pytest.raises(B.BfpError):
        B.Multigrid(cfg)
