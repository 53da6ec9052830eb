"""Golden fixtures of the BASELINE.json config solves at their FULL sizes.

TEST INFRASTRUCTURE: runs the C oracle (oracle/bfp_oracle.c, OpenMP; the
restatement of P/src/{wideint,bfp,blas}.cpp and the DESIGN.md section 3
driver of P/src/multigrid.cpp:399-518) on every config of FULL below and
records, per solve, the exact final iterate as a SHA-256 of its int64
little-endian mantissas in logical order (and per z-plane for 3-D), its
(q, e), the residual history (doubles from exact values, P/src/multigrid.cpp:480)
and a SHA-256 of the per-op trace.  tests/test_gpu_full_configs.py compares
the GPU solves with these fixtures bit for bit.

Run (this container: 8 cores, 62 GB; every case except C5 at 1023^3):
    python tests/golden/make_full_golden.py [--only NAME ...]
C5 at 1023^3 (about 60 GB of host memory for the oracle) is minted on the
GPU box host:  python tests/golden/make_full_golden.py --only C5_1023_p48
"""
import argparse
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

OUT = os.path.join(HERE, "full_configs.json")

PROG = [0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]  # C3: p_l = 4 + 2(l - 3)

# name -> solver config (paper_2307_00124_b200.mg_config / oracle.ob.mg_config keywords)
FULL = {
    "C1": dict(d=1, l_fine=20, cycles=10, x0_random=True, rhs_kind=0, p=16, pd=28, w_add_cap=4),
    "C2": dict(d=2, l_fine=12, cycles=15, rhs_kind=1, p=20),
    "C3": dict(d=2, l_fine=13, l_coarse=3, cycles=1, rhs_kind=1, fmg=True, nonnormalized=True,
               p=PROG),
    "C4": dict(d=3, l_fine=9, cycles=1, rhs_kind=1, fmg=True, p=24),
    "C4_n2": dict(d=3, l_fine=9, cycles=2, rhs_kind=1, fmg=True, p=24),
    "C4_v21_n2": dict(d=3, l_fine=9, cycles=2, rhs_kind=1, fmg=True, nu2=1, p=24),
    # the fastest variant below the discretisation error (tools/fmg_sweep2.py): V(2,0) x 2,
    # coarsest level 7^3 with 32 Jacobi sweeps
    "C4_v20_n2_lc3": dict(d=3, l_fine=9, l_coarse=3, cycles=2, rhs_kind=1, fmg=True, nu2=0,
                          n_coarse=32, p=24),
}
for _p in (4, 8, 16, 32, 48):
    FULL[f"C5_511_p{_p}"] = dict(d=3, l_fine=9, cycles=10, x0_random=True, rhs_kind=2, p=_p)
for _p in (4, 8, 16):
    FULL[f"C5_511_p{_p}_wdot24"] = dict(d=3, l_fine=9, cycles=10, x0_random=True, rhs_kind=2,
                                        p=_p, pd=24, w_add_cap=4)
FULL["C5_1023_p48"] = dict(d=3, l_fine=10, cycles=10, x0_random=True, rhs_kind=2, p=48)
BOX_ONLY = {"C5_1023_p48"}


def iterate_hashes(m, d, l):
    """(whole-array sha256, per-plane sha256 list or None) of int64 LE mantissas."""
    import numpy as np
    a = np.ascontiguousarray(m, dtype="<i8")
    whole = hashlib.sha256(a.tobytes()).hexdigest()
    planes = None
    if d == 3:
        n = (1 << l) - 1
        v = a.reshape(n, n * n)
        planes = [hashlib.sha256(v[k].tobytes()).hexdigest() for k in range(n)]
    return whole, planes


def trace_hash(trace):
    return hashlib.sha256(json.dumps([list(map(int, t)) for t in trace]).encode()).hexdigest()


def mint(name):
    from oracle import ob
    kw = dict(FULL[name])
    t0 = time.time()
    try:
        x, hist, tr = ob.mg_run(ob.mg_config(**kw), trace_cap=1 << 16)
    except ob.OracleError as ex:
        return {"config": kw, "oracle_error": str(ex)}
    whole, planes = iterate_hashes(x.m, kw["d"], kw["l_fine"])
    rec = {"config": kw, "x_q": x.q, "x_e": x.e, "x_sha256": whole, "history": hist,
           "n_trace": len(tr), "trace_sha256": trace_hash(tr),
           "recomputes": int(sum(t[8] for t in tr)), "oracle_s": round(time.time() - t0, 1)}
    if planes is not None and kw["l_fine"] >= 10:
        rec["plane_sha256"] = planes
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--out", default=OUT)
    a = ap.parse_args()
    names = a.only or [n for n in FULL if n not in BOX_ONLY]
    db = {}
    if os.path.exists(a.out):
        with open(a.out) as f:
            db = json.load(f)
    db.setdefault("_about", "oracle/bfp_oracle.c solves at BASELINE sizes; "
                            "made by tests/golden/make_full_golden.py")
    for n in names:
        rec = mint(n)
        db[n] = rec
        print(n, {k: v for k, v in rec.items() if k not in ("plane_sha256", "history")},
              flush=True)
        with open(a.out, "w") as f:
            json.dump(db, f, indent=1)


if __name__ == "__main__":
    main()
