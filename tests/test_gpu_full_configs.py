"""BASELINE.json configs 1-5 at their FULL sizes: the GPU solves against the oracle.

Every solve below runs on the device through the C-ABI (bfp_mg_create / bfp_mg_solve /
bfp_mg_result, graph-replayed) and must equal the C oracle (oracle/bfp_oracle.c, the
restatement of P/src/{wideint,bfp,blas}.cpp and the DESIGN.md section 3 driver of
P/src/multigrid.cpp:399-518) bit for bit:

* the final iterate (SHA-256 of its int64 mantissas, per z-plane at 1023^3), q and e;
* the residual history (doubles of exact norms, P/src/multigrid.cpp:480-482);
* the per-op trace (step, level, w_out, w_tmp, gamma, overflow, underflow, recompute,
  normalized; P/src/multigrid.cpp:157-170) through its SHA-256.

The oracle outputs are committed fixtures (tests/golden/full_configs.json, minted by
tests/golden/make_full_golden.py); test_c4_fmg_live_oracle also re-runs the oracle
live.  These sizes are the ones where the pipelined kernels run (2-D bulk pipeline and
row-march transfers at N >= 1024, 3-D tiled-TMA pipeline and plane-march transfers at
N >= 128): the kernel-family counters prove they were part of each checked solve.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from tests.golden.make_full_golden import FULL

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_configs.json")


def _fixtures():
    if not os.path.exists(GOLD):
        return {}
    with open(GOLD) as f:
        return json.load(f)


FIX = _fixtures()
NAMES = [n for n in FULL if n in FIX and "oracle_error" not in FIX[n]]

# kernel families each config's solve must exercise
MUST_RUN = {
    "C2": ("bulk2", "pro2", "rst2"),
    "C3": ("bulk2", "pro2", "rst2"),
    "C4": ("bulk3", "pro3", "rst3"),
    "C5": ("bulk3", "pro3", "rst3"),
}


def _sha(a):
    return hashlib.sha256(memoryview(np.ascontiguousarray(a, dtype="<i8"))).hexdigest()


def _trace_sha(tr):
    return hashlib.sha256(json.dumps([list(map(int, t)) for t in tr]).encode()).hexdigest()


def _solve(B, kw):
    kw = dict(kw)
    p = kw.pop("p")
    fam0 = B.kernel_family_counts()
    mg = B.Multigrid(B.mg_config(**kw, p=p))
    mg.solve(use_graph=True)
    out = mg.result(trace_cap=1 << 16)
    fam1 = B.kernel_family_counts()
    used = {k for k in fam1 if fam1[k] > fam0[k]}
    del mg
    return out, used


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_full_config_solve_vs_oracle(gpu, name):
    B = gpu
    rec = FIX[name]
    (x, q, e, hist, tr), used = _solve(B, rec["config"])
    assert (q, e) == (rec["x_q"], rec["x_e"]), name
    kw = rec["config"]
    if "plane_sha256" in rec:  # 1023^3: locate a mismatch by z-plane
        n = (1 << kw["l_fine"]) - 1
        v = x.reshape(n, n * n)
        bad = [k for k in range(n) if _sha(v[k]) != rec["plane_sha256"][k]]
        assert not bad, f"{name}: planes {bad[:8]} differ"
    assert _sha(x) == rec["x_sha256"], name
    assert hist == rec["history"], name
    assert len(tr) == rec["n_trace"] and _trace_sha(tr) == rec["trace_sha256"], name
    for fam in MUST_RUN.get(name.split("_")[0], ()):
        assert fam in used, f"{name}: kernel family {fam} not used ({sorted(used)})"


@pytest.mark.gpu
def test_c4_fmg_live_oracle(gpu):
    """Config 4 (511^3 FMG, p = 24) against the oracle run live on the host: every
    mantissa, the history and every trace record."""
    from oracle import ob
    B = gpu
    kw = dict(FULL["C4"])
    ox, oh, otr = ob.mg_run(ob.mg_config(**kw), trace_cap=1 << 16)
    (x, q, e, hist, tr), _ = _solve(B, kw)
    assert (q, e) == (ox.q, ox.e)
    assert np.array_equal(x, ox.m)
    assert hist == oh
    assert [tuple(t) for t in tr] == [tuple(t) for t in otr]


def test_fixtures_cover_the_configs():
    """CPU check: the committed fixtures cover configs 1-5 (C5 at 511^3 for every p and
    at 1023^3 for p = 48) and name the solver config they were minted with."""
    for n in ("C1", "C2", "C3", "C4", "C4_v21_n2"):
        assert n in FIX, n
    for p in (4, 8, 16, 32, 48):
        assert f"C5_511_p{p}" in FIX, p
    for n, rec in FIX.items():
        if n.startswith("_"):
            continue
        assert rec["config"] == FULL[n], n
