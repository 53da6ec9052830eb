#!/usr/bin/env python
"""Benchmark of the B200 BFP multigrid hot path (BASELINE.json metric).

Metric: "BFP stencil residual GDoF/s + % of HBM roofline; FMG solve time to disc.
accuracy".  BASELINE.json names no config for it, so the N = 1 line is quoted on the
largest single-GPU config, config 4:

`value`: BFP stencil residual throughput in GDoF/s on config 4's fine level --
r = b - A x, 3-D 7-point, 511^3 interior, int32 mantissas p = 24, qcomp window
(w_tmp = p + 5), exact int64 accumulation -- with inputs resident in HBM (two
(x, b, r) sets of 1.6 GB each, far above the 126 MB L2).  One step = one windowed
residual over the whole grid (pass 1 + the recompute launch, which exits early on the
fast path).

`roofline`: the dominant kernel (pass 1 of the residual, bulk3_win_kernel) timed with
CUDA events on its launch stream over a fixed loop of 200 launches (independent of
--steps), 12 algorithmic bytes per DoF, against MEASURED_PEAKS.json.
`e2e`: the same metric through the C-ABI with HOST buffers: every step uploads x and b
(int32, pinned) and downloads r, copies inside the timed region.
`cpu_baseline`: the CPU oracle port (oracle/bfp_oracle.c, OpenMP, all host threads) on
the same residual, a single-thread sample, and the FMG solve to discretisation accuracy
(config 4, two IR-V(2,1) per level) on the host cores.
`solves`: device time of the config solves (C1-C5) replayed as CUDA graphs, each with
its algorithmic-bytes roofline fraction and accuracy; `summary` (last key) repeats the
numbers a reader needs in a few hundred bytes.

`--impl reference` times the reference's CPU path (the oracle port of P/src/blas.cpp
qcomp + EgemvKernel; the GMP reference itself cannot be built here) on
the same config and metric.  `--gpus N` without torchrun spawns its own N ranks.
"""
import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

D, L_FINE, P_BITS = 3, 9, 24  # config 4's fine level
W_TMP = P_BITS + 5
N_SETS = 2
BYTES_PER_DOF = 12  # x, b read once + r written once, int32
KERNEL_LAUNCHES = 200  # fixed pass-1 loop of the roofline timing


def dof(d=D, l=L_FINE):
    return ((1 << l) - 1) ** d


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        try:
            out, _ = self.p.communicate(timeout=5)
        except Exception:
            self.p.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [t.strip() for t in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(n):
    """`bench.py --gpus N` outside torchrun: start N ranks of this script (one per GPU,
    env rendezvous on 127.0.0.1) and return the worst exit code; rank 0 prints the line."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n),
                   LOCAL_WORLD_SIZE=str(n), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:],
                                      env=env))
    return max(p.wait() for p in procs)


# ---------------------------------------------------------------------------
# CPU side (test-infrastructure oracle, oracle/bfp_oracle.c): the reference arm and the
# cpu_baseline legs


def cpu_inputs(d, l, p):
    from oracle import ob
    x = ob.gen_uniform(d, l, p, 1, 1)
    b = ob.gen_uniform(d, l, p, 1, 2) if d == 1 else ob.gen_sine(d, l, p)
    return x, b


def cpu_residual_time(steps, warmup, budget_s=None, threads=None, d=D, l=L_FINE, p=P_BITS):
    """The oracle's OpenMP qcomp residual on the workload's inputs (all host threads, or
    `threads`). Returns (seconds per residual, threads, residuals run)."""
    from oracle import ob
    L = ob.lib()
    x, b = cpu_inputs(d, l, p)
    out = ob.OBlock(x.m.copy(), p, 0)
    xc, bc, oc = x.c(), b.c(), out.c()
    fl = ob.Flags()
    threads = threads or os.cpu_count() or 1
    g = ob.Grid(d, l)
    gm, ge = 1 << 14, 2 * l + 8
    rc = L.ob_residual_qcomp_omp(g, C.byref(xc), C.byref(bc), p, p + 5, gm, ge, C.byref(oc),
                                 C.byref(fl), threads)
    assert rc == 0
    # exact-binade gamma: the qcomp fast path, as on the GPU
    mx = int(abs(out.m).max()) if len(out.m) else 0
    ge = oc.e + mx.bit_length() + 1 - 16 if mx else 0
    for _ in range(warmup):
        L.ob_residual_qcomp_omp(g, C.byref(xc), C.byref(bc), p, p + 5, gm, ge, C.byref(oc),
                                C.byref(fl), threads)
    t0 = time.perf_counter()
    n = 0
    while n < steps:
        L.ob_residual_qcomp_omp(g, C.byref(xc), C.byref(bc), p, p + 5, gm, ge, C.byref(oc),
                                C.byref(fl), threads)
        n += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    return (time.perf_counter() - t0) / n, threads, n


def cpu_fmg_time(name):
    """Wall time of one config solve on the host cores (oracle, OpenMP, all threads)."""
    from oracle import ob
    kw = dict(SOLVES[name])
    t0 = time.perf_counter()
    x, hist, tr = ob.mg_run(ob.mg_config(**kw), trace_cap=1 << 16)
    return time.perf_counter() - t0, hist[-1], len(tr)


def host_cpu():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip() + f" ({os.cpu_count()} threads)"
    except OSError:
        pass
    return f"{os.cpu_count()} threads"


def traffic_bytes(args):
    """ncu dram read + write bytes per pass-1 launch of the dominant kernel, from the
    committed capture (profiles/r2_traffic.json) unless given on the command line."""
    if args.traffic_bytes is not None:
        return args.traffic_bytes
    try:
        with open(os.path.join(REPO, "profiles", "r2_traffic.json")) as f:
            return json.load(f)["c4_residual_pass1"]["traffic_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def workload_config(world=1):
    return {"workload": "BASELINE config 4 fine-level BFP residual r=b-A*x (3-D 7-point, "
                        "511^3 interior, int32 mantissas p=24, qcomp w_tmp=29, exact int64 "
                        "accumulation)",
            "dof": dof(), "bytes_per_dof": BYTES_PER_DOF,
            "l2": f"inputs above L2: {N_SETS} (x,b,r) sets of {3 * 4 * dof() / 1e9:.2f} GB "
                  "(126 MB L2), alternated per step",
            "parallelism": "single GPU" if world == 1 else f"z-slab x{world}"}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    sec, threads, n = cpu_residual_time(args.steps, args.warmup)
    v = dof() / sec / 1e9
    line = {
        "impl": "reference", "metric": "bfp_stencil_residual_gdofs", "value": v, "unit": "GDoF/s",
        "n_gpus": 0, "steps": n, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
        "data": "synthetic", "config": workload_config(),
        "cpu_baseline": {"value": v, "unit": "GDoF/s", "cores": threads, "kind": "port",
                         "sample": f"{n} full 511^3 residuals (oracle/bfp_oracle.c OpenMP; the "
                                   "GMP reference is unbuildable here)",
                         "host_cpu": host_cpu()},
        "e2e": {"value": v, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def solve_bytes(trace, d, s):
    """Algorithmic HBM bytes of a solve from its trace: per op the bytes of each operand
    read once + the output written once: residual / Jacobi / axpby 3s,
    first sweep 2s, restriction and FMG prolongation (1 + 2^-d)s, prolong + correct
    (2 + 2^-d)s per fine DoF of the op's level."""
    per = {0: 3, 1: 3, 2: 2, 3: 3, 4: 3, 5: 1 + 2.0 ** -d, 6: 2 + 2.0 ** -d, 7: 1 + 2.0 ** -d,
           8: 3}
    return sum(per[t[0]] * s * ((1 << t[1]) - 1) ** d for t in trace)


def run_ours(args, world, rank, local):
    import torch
    torch.cuda.set_device(local)
    import paper_2307_00124_b200 as B
    stream = torch.cuda.current_stream()
    B.set_stream(stream.cuda_stream)
    Lb = B.lib()
    sp = C.c_void_p(stream.cuda_stream)
    n = dof()

    # inputs resident in HBM: N_SETS independent (x, b, r), each set 1.6 GB (> L2)
    xs, bs, rs, gs = [], [], [], []
    for s in range(N_SETS):
        x = B.gen_uniform(B.BfpVec.grid(D, L_FINE, 4), P_BITS, 1 + s + 100 * rank, 1)
        b = B.gen_sine(B.BfpVec.grid(D, L_FINE, 4), P_BITS)
        r = B.BfpVec.grid(D, L_FINE, 4)
        # gamma with the exact binade of the residual: the qcomp fast path (Table 2 regime)
        B.residual(x, b, P_BITS, W_TMP, B.Scalar(1 << 14, 16, 2 * L_FINE + 8), out=r)
        gs.append(B.inf_norm_upper(r))
        xs.append(x)
        bs.append(b)
        rs.append(r)
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()

    def step(k):
        s = k % N_SETS
        rc = Lb.bfp_stencil_gemv(xs[s].h, bs[s].h, m1, p1, 0, P_BITS, W_TMP, gs[s].c(), 0,
                                 rs[s].h, sp)
        if rc:
            raise RuntimeError(f"bfp_stencil_gemv failed: {rc}")

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    torch.cuda.synchronize()
    l0 = B.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = B.launch_count() - l0
    ms = e0.elapsed_time(e1)
    # dominant-kernel time: pass 1 alone over a fixed loop of KERNEL_LAUNCHES launches (the
    # recompute launch is skipped; valid because gamma has the exact binade, checked
    # below), CUDA events on the launch stream around the whole loop
    B.set_kernel_path(skip_recompute=True)
    for k in range(4):
        step(k)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for k in range(KERNEL_LAUNCHES):
        step(k)
    k1.record(stream)
    torch.cuda.synchronize()
    B.set_kernel_path()
    clk = clocks.stop()
    kern_ms = k0.elapsed_time(k1)
    for r_ in rs:
        assert not (r_.header().flags & B.FLAG_RECOMPUTED), "recompute needed: pass-1 timing invalid"
    # per-launch event brackets (serialising; secondary evidence)
    B.profile_enable(True)
    B.profile_read(reset=True)
    for k in range(50):
        step(k)
    torch.cuda.synchronize()
    ev_ms, ev_n = B.profile_read(reset=True)
    B.profile_enable(False)
    value = n * args.steps / (ms / 1e3) / 1e9
    hdr = rs[0].header()
    assert hdr.err == 0, "device error in timed residuals"

    peak, peak_kind = peaks()
    kavg_ms = kern_ms / KERNEL_LAUNCHES
    achieved = BYTES_PER_DOF * n / (kavg_ms / 1e3) / 1e9
    tb = traffic_bytes(args)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": tb,
            "kernel": "bulk3_win_kernel<QCOMP,int32,GemvOp> pass 1 (tiled-TMA plane march)",
            "peak_kind": peak_kind, "kernel_ms": kavg_ms,
            "kernel_ms_event_brackets": ev_ms / max(ev_n, 1),
            "timing": f"pass 1 back to back, {KERNEL_LAUNCHES} launches (fixed, independent of "
                      "--steps), recompute skipped (flags verified clear), CUDA events on the "
                      "launch stream around the loop",
            "algorithmic_bytes_per_launch": BYTES_PER_DOF * n,
            "traffic_source": "profiles/r2_traffic.json (ncu --set full, same kernel)"}
    del xs, bs, rs
    clean(torch)

    e2e = run_e2e(args, B, Lb, torch, stream, sp, D, L_FINE, P_BITS)
    clean(torch)

    line = {
        "metric": "bfp_stencil_residual_gdofs", "value": value, "unit": "GDoF/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic", "config": workload_config(),
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
    }
    if not args.no_extras:
        # kernel-level numbers first, each section from a clean allocator state
        line["residual_other_configs"] = {
            "C2_2d_4095^2_int32_p20": measure_residual(B, torch, stream, 2, 12, 20, 4, steps=100),
            "C1_1d_2^20_int32_p16": measure_residual(B, torch, stream, 1, 20, 16, 4, steps=200),
            # config 1 is L2-resident; the %HBM claim for 1-D needs n beyond L2
            "C1_1d_2^28_int32_p16_probe": measure_residual(B, torch, stream, 1, 28, 16, 4,
                                                           steps=20),
            "C5_3d_1023^3_int64_p48": measure_residual(B, torch, stream, 3, 10, 48, 8, steps=20),
        }
        clean(torch)
        line["fine_level_ops"] = {"C4": measure_ops(B, torch, stream, 3, 9, 24),
                                  "C2": measure_ops(B, torch, stream, 2, 12, 20),
                                  "C5": measure_ops(B, torch, stream, 3, 10, 48, steps=10, s=8)}
        clean(torch)
        line["solves"] = run_solves(B, torch, stream)
        ttd = {k: v for k, v in line["solves"].items()
               if v.get("accuracy", {}).get("alg_over_disc", 1e30) <= 1.0}
        if ttd:
            k = min(ttd, key=lambda k: ttd[k]["ms"])
            line["fmg_time_to_disc_accuracy"] = {
                "config": k, "ms": ttd[k]["ms"],
                "alg_over_disc": ttd[k]["accuracy"]["alg_over_disc"],
                "note": "max-norm error vs the discrete solution <= the discretisation error"}
        clean(torch)
        line["C5_precision_sweep_1gpu"] = run_c5_sweep(B, torch, stream)
    if not args.no_cpu:
        sec, threads, nrun = cpu_residual_time(10**9, 1, budget_s=args.cpu_budget)
        sec1, _, nrun1 = cpu_residual_time(10**9, 0, budget_s=args.cpu_budget / 2, threads=1)
        cb = {"value": n / sec / 1e9, "unit": "GDoF/s", "cores": threads, "kind": "port",
              "sample": f"{nrun} full 511^3 residuals in ~{args.cpu_budget:.0f} s "
                        "(oracle/bfp_oracle.c, OpenMP)",
              "single_thread": {"value": n / sec1 / 1e9, "cores": 1,
                                "sample": f"{nrun1} full 511^3 residuals, one thread (the "
                                          "reference's loops are sequential)"},
              "host_cpu": host_cpu()}
        if not args.no_cpu_fmg:
            name = line.get("fmg_time_to_disc_accuracy", {}).get("config", "C4_3d_fmg_v21_n2")
            t, fres, nops = cpu_fmg_time(name)
            cb["fmg_solve"] = {"config": name, "s": t, "cores": threads, "ops": nops,
                               "final_residual": fres,
                               "sample": "one full solve (oracle mg_run, OpenMP)"}
        line["cpu_baseline"] = cb
    line["summary"] = summary(line)
    print(json.dumps(line), flush=True)
    return 0


def summary(line):
    """The numbers a reader needs, compact, as the LAST key of the line."""
    r = lambda v, k=3: None if v is None else round(v, k)  # noqa: E731
    s = {"C4_residual": {"gdofs": r(line["value"], 1), "hbm_frac": r(line["roofline"]["frac"]),
                         "e2e_gdofs": r(line["e2e"]["value"], 2)}}
    for k, v in line.get("residual_other_configs", {}).items():
        if "hbm_frac" in v:
            s[k.split("_")[0] + ("_probe" if "probe" in k else "")] = r(v["hbm_frac"])
    ops = line.get("fine_level_ops", {})
    for c in ("C4", "C2", "C5"):
        if c in ops:
            s[c + "_ops_frac"] = {k: r(v["hbm_frac"], 2) for k, v in ops[c]["ops"].items()}
    sol = line.get("solves", {})
    s["solves_ms"] = {k.split("_")[0] + k[k.find("_fmg"):] if "_fmg" in k else k.split("_")[0]:
                      [r(v.get("ms"), 2), r(v.get("hbm_frac"), 2)]
                      for k, v in sol.items() if "ms" in v}
    t = line.get("fmg_time_to_disc_accuracy")
    cb = line.get("cpu_baseline", {})
    if t:
        s["fmg_to_disc"] = {"gpu_ms": r(t["ms"], 2), "cfg": t["config"]}
        if "fmg_solve" in cb:
            s["fmg_to_disc"]["cpu_s"] = r(cb["fmg_solve"]["s"], 2)
            s["fmg_to_disc"]["cpu_cores"] = cb["fmg_solve"]["cores"]
    c5 = line.get("C5_precision_sweep_1gpu", {})
    if c5:
        s["C5_sweep_ms"] = {k: r(v.get("ms"), 1) for k, v in c5.items()}
    if cb:
        s["cpu_residual_gdofs"] = r(cb.get("value"))
    return s


def run_e2e(args, B, Lb, torch, stream, sp, d, l, p):
    """Same metric through the C-ABI with pinned HOST buffers, pipelined across steps:
    stream A[k%2] uploads x, b (one contiguous H2D copy each into a staging buffer + a scatter
    kernel into the padded layout) and runs
    the residual into buffer k%2; stream B downloads r of step k (gather + D2H engine)
    while A[(k+1)%2] uploads step k+1 (H2D engine).  `pcie_h2d_gbs`: one step's H2D bytes
    copied alone (the bound of this arm)."""
    n = dof(d, l)
    x = B.gen_uniform(B.BfpVec.grid(d, l, 4), p, 1, 1)
    b = B.gen_sine(B.BfpVec.grid(d, l, 4), p)
    hx = torch.empty(n, dtype=torch.int32).pin_memory()
    hb = torch.empty(n, dtype=torch.int32).pin_memory()
    hr = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
    hh = B._Header()
    for src, dst in ((x, hx), (b, hb)):
        assert Lb.bfp_vec_download_i32(src.h, C.c_void_p(dst.data_ptr()), C.byref(hh), sp) == 0
    qx, ex = x.q, x.e
    qb, eb = b.q, b.e
    del x, b
    xd = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    bd = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    rd = [B.BfpVec.grid(d, l, 4) for _ in range(2)]
    Lb.bfp_vec_upload_i32(xd[0].h, C.c_void_p(hx.data_ptr()), qx, ex, sp)
    Lb.bfp_vec_upload_i32(bd[0].h, C.c_void_p(hb.data_ptr()), qb, eb, sp)
    B.residual(xd[0], bd[0], p, p + 5, B.Scalar(1 << 14, 16, 2 * l + 8), out=rd[0])
    g = B.inf_norm_upper(rd[0]).c()
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()
    sas = [stream, torch.cuda.Stream()]
    sa = stream
    sb = torch.cuda.Stream()
    pas = [C.c_void_p(s_.cuda_stream) for s_ in sas]
    pb = C.c_void_p(sb.cuda_stream)
    ev_r = [torch.cuda.Event() for _ in range(2)]
    ev_d = [torch.cuda.Event() for _ in range(2)]
    for e in ev_d:
        e.record(sb)

    def step(k):
        i = k & 1
        sa, pa = sas[i], pas[i]
        sa.wait_event(ev_d[i])  # download of step k-2 finished with rd[i]
        assert Lb.bfp_vec_upload_i32(xd[i].h, C.c_void_p(hx.data_ptr()), qx, ex, pa) == 0
        assert Lb.bfp_vec_upload_i32(bd[i].h, C.c_void_p(hb.data_ptr()), qb, eb, pa) == 0
        assert Lb.bfp_stencil_gemv(xd[i].h, bd[i].h, m1, p1, 0, p, p + 5, g, 0, rd[i].h,
                                   pa) == 0
        ev_r[i].record(sa)
        sb.wait_event(ev_r[i])
        assert Lb.bfp_vec_download_async_i32(rd[i].h, C.c_void_p(hr[i].data_ptr()), pb) == 0
        ev_d[i].record(sb)

    k = max(3, min(args.steps, 20))
    for j in range(2):
        step(j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(sa)
    sas[1].wait_stream(sa)
    for j in range(k):
        step(j)
    sa.wait_stream(sb)
    sa.wait_stream(sas[1])
    e1.record(sa)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # the PCIe bound: one step's H2D bytes (x and b) alone, pinned, same engine
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dx = torch.empty(n, dtype=torch.int32, device="cuda")
    db = torch.empty(n, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(sa):
        for _ in range(2):
            dx.copy_(hx, non_blocking=True)
        h0.record(sa)
        for _ in range(3):
            dx.copy_(hx, non_blocking=True)
            db.copy_(hb, non_blocking=True)
        h1.record(sa)
    torch.cuda.synchronize()
    h2d_gbs = 3 * 2 * 4 * n / (h0.elapsed_time(h1) / 1e3) / 1e9
    h = rd[(k - 1) & 1].header()
    assert h.err == 0
    return {"value": n * k / (ms / 1e3) / 1e9, "unit": "GDoF/s", "h2d_bytes_per_step": 2 * 4 * n,
            "d2h_bytes_per_step": 4 * n, "steps": k, "ms_per_step": ms / k,
            "pcie_h2d_gbs": h2d_gbs, "pcie_bound_frac": 2 * 4 * n / (ms / k / 1e3) / 1e9 / h2d_gbs,
            "path": "bfp_vec_upload_i32 x2 + bfp_stencil_gemv (streams A0/A1 by step parity) | "
                    "bfp_vec_download_async_i32 (stream B), pinned host, double-buffered"}


def run_sharded(args, world, rank, local):
    """N GPUs: config 4's fine-level residual z-slab sharded over the ranks (strong
    scaling: the 511^3 grid is fixed, each rank owns 512/N planes) through the native
    sharded op (bfp_dist_stencil_gemv: NCCL halo exchange of one plane per neighbour,
    partial windows, MAX all-reduces, finalize -- all enqueued on the stream, no host
    synchronisation).  Two slab sets alternate per step (per-rank bytes stay above the
    L2 at every N <= 8).  The line also carries the sharded config-4 FMG solve (the
    metric's second half) and config 5's precision sweep on 1023^3 z-slabs.
    --sharded forces this path at N = 1."""
    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    import paper_2307_00124_b200 as B
    from paper_2307_00124_b200 import dist as Dm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    B.set_stream(stream.cuda_stream)
    n = dof()
    nn_ = (1 << L_FINE) - 1
    per = nn_ * nn_
    lo, hi = Dm.slab_ranges(L_FINE, world)[rank]

    def make_ops():
        idt = torch.zeros(B.NCCL_ID_BYTES, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(B.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        return B.DistOps(world, rank, bytes(idt.cpu().numpy().tobytes()))

    ops = make_ops()
    transport = "default (peer-memory mailboxes when CUDA IPC maps them, else ncclAllReduce)"

    sets = []
    for s in range(N_SETS):
        gx = B.gen_uniform(B.BfpVec.grid(D, L_FINE, 4), P_BITS, 1 + s, 1)
        gb = B.gen_sine(B.BfpVec.grid(D, L_FINE, 4), P_BITS)
        g = B.inf_norm_upper(B.residual(gx, gb, P_BITS, W_TMP,
                                        B.Scalar(1 << 14, 16, 2 * L_FINE + 8)).z)

        def slab_of(full):
            m, q, e = full.download()
            v = B.BfpVec.slab(D, L_FINE, lo, hi)
            v.upload(m[lo * per: min(hi, nn_) * per], q, e)
            return v
        sets.append((slab_of(gx), slab_of(gb), B.BfpVec.slab(D, L_FINE, lo, hi), g))
        if s == 0:
            ref0 = B.residual(gx, gb, P_BITS, W_TMP, g).z.download()
        del gx, gb
    clean(torch)
    m1, p1 = B.bfp_minus_one(), B.bfp_one()

    def step(k):
        xs, bs, rr, g = sets[k % N_SETS]
        ops.gemv([xs], [bs], m1, p1, P_BITS, W_TMP, g, [rr])

    def parity_ok():
        """set 0's sharded residual equals the unsharded one on this rank's planes, on every rank"""
        okl = 0
        try:
            step(0)
            mo, _, eo = sets[0][2].download()
            mr, _, er = ref0
            okl = int(eo == er and np.array_equal(mo, mr[lo * per: min(hi, nn_) * per]))
        except Exception as ex:  # noqa: BLE001 -- a transport error surfaces as a status
            print(f"[bench] rank {rank}: sharded step failed: {ex}", file=sys.stderr)
        okt = torch.tensor([okl], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        return bool(okt.item())

    # Self-check of the exponent all-reduce transport before anything is timed: the mailbox
    # protocol is bit-exact in the in-process tests, but this is the first use on this box's
    # peer mappings -- on any mismatch fall back to ncclAllReduce and say so in the line.
    if not parity_ok():
        del ops
        B.set_transport(2)
        ops = make_ops()
        transport = "ncclAllReduce (mailbox self-check failed on this box)"
    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = B.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        step(k)
    e1.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = B.launch_count() - l0
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # parity of set 0's sharded residual with the unsharded one on this rank's planes
    sharded_ok = parity_ok()
    peak, peak_kind = peaks()
    achieved = BYTES_PER_DOF * n / world / (ms / args.steps / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
            "timing": "per-GPU share of the algorithmic bytes over the whole sharded step "
                      "(halo + pass 1 + all-reduces + finalize), max over ranks"}
    e2e = sharded_e2e(B, torch, dist, stream, ops, world, rank, lo, hi, args)
    del sets
    clean(torch)
    solve = {} if args.no_extras else sharded_solve(B, torch, dist, stream, world, rank)
    clean(torch)
    c5 = {} if args.no_extras else sharded_c5_sweep(B, torch, dist, stream, world, rank)
    line = {
        "metric": "bfp_stencil_residual_gdofs", "value": n * args.steps / (ms / 1e3) / 1e9,
        "unit": "GDoF/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": dict(workload_config(world),
                       parallelism=f"z-slab x{world} (NCCL halo + MAX allreduce)"),
        "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk,
        "sharded_parity_with_unsharded": sharded_ok, "exponent_allreduce_transport": transport,
        "sharded_solve_C4": solve, "C5_precision_sweep_sharded": c5,
    }
    if rank == 0 and not args.no_cpu:
        sec, threads, nrun = cpu_residual_time(10**9, 1, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": n / sec / 1e9, "unit": "GDoF/s", "cores": threads,
                                "kind": "port", "host_cpu": host_cpu(),
                                "sample": f"{nrun} full 511^3 residuals (oracle, OpenMP)"}
    dist.barrier()
    del ops
    dist.destroy_process_group()
    if rank == 0:
        line["summary"] = {"C4_residual_gdofs": round(line["value"], 1),
                           "per_gpu_hbm_frac": round(roof["frac"], 3),
                           "e2e_gdofs": round(e2e.get("value", 0.0), 2),
                           "C4_fmg_ms": solve.get("ms"),
                           "C5_sweep_ms": {k: v.get("ms") for k, v in c5.items()}}
        print(json.dumps(line), flush=True)
    return 0


def sharded_e2e(B, torch, dist, stream, ops, world, rank, lo, hi, args):
    """The sharded residual through the C-ABI with pinned HOST buffers, pipelined like the
    one-GPU arm (run_e2e): every step each rank uploads its x and b slabs (int32, pinned;
    stream A, followed by the sharded op on the same stream) while stream B gathers and
    downloads the previous step's r slab; two buffer sets alternate.  Every rank drives its
    own PCIe link, so the arm scales with N.  Device time (CUDA events on stream A after
    joining B), max over ranks."""
    import numpy as np
    nn_ = (1 << L_FINE) - 1
    per = nn_ * nn_
    try:
        Lb = B.lib()
        gx = B.gen_uniform(B.BfpVec.grid(D, L_FINE, 4), P_BITS, 1, 1)
        gb = B.gen_sine(B.BfpVec.grid(D, L_FINE, 4), P_BITS)
        g = B.inf_norm_upper(B.residual(gx, gb, P_BITS, W_TMP,
                                        B.Scalar(1 << 14, 16, 2 * L_FINE + 8)).z)
        (mx_, qx, ex), (mb_, qb, eb) = gx.download(), gb.download()
        del gx, gb
        sl = slice(lo * per, min(hi, nn_) * per)
        hx = torch.from_numpy(np.ascontiguousarray(mx_[sl]).astype(np.int32)).pin_memory()
        hb = torch.from_numpy(np.ascontiguousarray(mb_[sl]).astype(np.int32)).pin_memory()
        del mx_, mb_
        nloc = hx.numel()
        hr = [torch.empty(nloc, dtype=torch.int32).pin_memory() for _ in range(2)]
        xs = [B.BfpVec.slab(D, L_FINE, lo, hi) for _ in range(2)]
        bs = [B.BfpVec.slab(D, L_FINE, lo, hi) for _ in range(2)]
        rr = [B.BfpVec.slab(D, L_FINE, lo, hi) for _ in range(2)]
        m1, p1 = B.bfp_minus_one(), B.bfp_one()
        sa, sb = stream, torch.cuda.Stream()
        pa, pb = C.c_void_p(sa.cuda_stream), C.c_void_p(sb.cuda_stream)
        ev_r = [torch.cuda.Event() for _ in range(2)]
        ev_d = [torch.cuda.Event() for _ in range(2)]
        for e in ev_d:
            e.record(sb)

        def step(k):
            i = k & 1
            sa.wait_event(ev_d[i])  # the download of step k-2 is done with rr[i]
            assert Lb.bfp_vec_upload_i32(xs[i].h, C.c_void_p(hx.data_ptr()), qx, ex, pa) == 0
            assert Lb.bfp_vec_upload_i32(bs[i].h, C.c_void_p(hb.data_ptr()), qb, eb, pa) == 0
            ops.gemv([xs[i]], [bs[i]], m1, p1, P_BITS, W_TMP, g, [rr[i]])  # on stream A
            ev_r[i].record(sa)
            sb.wait_event(ev_r[i])
            assert Lb.bfp_vec_download_async_i32(rr[i].h, C.c_void_p(hr[i].data_ptr()), pb) == 0
            ev_d[i].record(sb)

        for j in range(2):
            step(j)
        k = max(3, min(args.steps, 20))
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sa)
        for j in range(k):
            step(j)
        sa.wait_stream(sb)
        e1.record(sa)
        torch.cuda.synchronize()
        assert rr[(k - 1) & 1].header().err == 0
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item()) / k
        return {"value": dof() / (ms / 1e3) / 1e9, "unit": "GDoF/s",
                "h2d_bytes_per_step": 2 * 4 * nloc, "d2h_bytes_per_step": 4 * nloc,
                "steps": k, "ms_per_step": ms,
                "path": "per rank: bfp_vec_upload_i32 x2 + bfp_dist_stencil_gemv (stream A) | "
                        "bfp_vec_download_async_i32 (stream B), pinned host, double-buffered; "
                        "bytes per rank, max over ranks"}
    except Exception as ex:  # noqa: BLE001 -- report, never hide
        return {"error": str(ex)}


def sharded_c5_sweep(B, torch, dist, stream, world, rank, ps=(4, 8, 16, 32, 48)):
    """Config 5 on the N ranks: 1023^3 z-slabs, x0 uniform, b = 0, 10 IR-V(2,2) per p
    (native sharded solver, one CUDA graph per solve); device time, max over ranks."""
    out = {}
    for p in ps:
        try:
            # one NCCL unique id per communicator (an id serves one ncclCommInitRank round)
            idt = torch.zeros(B.NCCL_ID_BYTES, dtype=torch.uint8, device="cuda")
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(B.nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nid = bytes(idt.cpu().numpy().tobytes())
            cfg = B.mg_config(d=3, l_fine=10, cycles=10, x0_random=True, rhs_kind=2, p=p)
            mg = B.Multigrid(cfg, world=world, rank=rank, nccl_id=nid, min_planes=16)
            mg.solve(use_graph=False)
            torch.cuda.synchronize()
            mg.solve(use_graph=True)
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mg.solve(use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1)], device="cuda", dtype=torch.float64)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
            out[f"p{p}"] = {"ms": float(ms.item()), "final_residual": hist[-1],
                            "first_residual": hist[0]}
            del mg
            clean(torch)
        except Exception as ex:  # noqa: BLE001 -- report, never hide
            out[f"p{p}"] = {"error": str(ex)}
    return out


def sharded_solve(B, torch, dist, stream, world, rank, name="C4_3d_fmg", min_planes=16, reps=3):
    """The C4 FMG solve with its fine levels z-slab sharded over the ranks (native
    solver, NCCL halo / MAX all-reduce / all-gather inside the plan, one CUDA graph per
    solve); strong scaling.  Parity: this rank's slab of the final iterate and the
    residual history equal the unsharded solve's."""
    import numpy as np
    kw = dict(SOLVES[name])
    cfg = B.mg_config(**kw)
    out = {"config": name, "min_planes": min_planes}
    try:
        idt = torch.zeros(B.NCCL_ID_BYTES, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(B.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
        mg = B.Multigrid(cfg, world=world, rank=rank, nccl_id=nid, min_planes=min_planes)
        mg.solve(use_graph=False)  # connections + first run outside capture
        torch.cuda.synchronize()
        graph = True
        try:
            mg.solve(use_graph=True)
        except Exception as ex:  # noqa: BLE001 -- report and time stream-ordered
            graph, out["graph_error"] = False, str(ex)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            mg.solve(use_graph=graph)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / reps], device="cuda", dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
        xv, rv, rk, ls = mg.rank_result(0)
        mx, _, ex_ = xv.download()
        ref = B.Multigrid(cfg)
        ref.solve(use_graph=True)
        xr, qr, er, hr, trr = ref.result(trace_cap=1 << 16)
        nn_ = (1 << cfg.l_fine) - 1
        per = nn_ ** (cfg.d - 1)
        lo = rank * ((1 << cfg.l_fine) // world) if ls <= cfg.l_fine else 0
        ok = ex_ == er and hist == hr and tr == trr and np.array_equal(
            mx, xr[lo * per: lo * per + len(mx)])
        okt = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        out.update(ms=float(ms.item()), graph=graph, lowest_sharded_level=ls,
                   parity_with_unsharded=bool(okt.item()), final_residual=hist[-1])
        del mg, ref
    except Exception as ex:  # noqa: BLE001 -- report, never hide
        out["error"] = str(ex)
    return out



def measure_residual(B, torch, stream, d, l, p, mb, steps=30):
    """Residual throughput on another config's fine level (inputs resident, qcomp with the
    exact-binade gamma; pass 1 alone timed back to back for the kernel time)."""
    sp = C.c_void_p(stream.cuda_stream)
    Lb = B.lib()
    x = B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 1, 1)
    # config 1's right-hand side is uniform (stream 2); the others are the sine rhs
    b_ = (B.gen_uniform(B.BfpVec.grid(d, l, mb), p, 1, 2) if d == 1 else
          B.gen_sine(B.BfpVec.grid(d, l, mb), p))
    r = B.BfpVec.grid(d, l, mb)
    B.residual(x, b_, p, p + 5, B.Scalar(1 << 14, 16, 2 * l + 8), out=r)
    g = B.inf_norm_upper(r).c()
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()
    n = ((1 << l) - 1) ** d

    def run(k):
        for _ in range(k):
            assert Lb.bfp_stencil_gemv(x.h, b_.h, m1, p1, 0, p, p + 5, g, 0, r.h, sp) == 0
    run(3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / steps
    B.set_kernel_path(skip_recompute=True)
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    B.set_kernel_path()
    kern_ms = e0.elapsed_time(e1) / steps
    assert not (r.header().flags & B.FLAG_RECOMPUTED)
    peak, _ = peaks()
    return {"dof": n, "mant_bytes": mb, "p": p, "gdofs": n / (step_ms / 1e3) / 1e9,
            "kernel_ms": kern_ms, "hbm_frac": 3 * mb * n / (kern_ms / 1e3) / 1e9 / peak}


def clean(torch):
    """Free the previous section's vectors (library handles die with their Python objects)."""
    import gc
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def measure_ops(B, torch, stream, d, l, p, steps=20, only=None, s=4):
    """Every fine-level op of the V-cycle / FMG on one config's finest level (inputs
    resident, gamma at the exact binade so qcomp takes the fast path): pass-1 kernel
    time (recompute launch skipped, flags verified) and its fraction of the measured
    HBM peak for the op's algorithmic bytes (residual / Jacobi / axpby
    3s, scal 2s, restriction (1 + 2^-d)s and prolongation (2^-d + 1)s per fine DoF,
    prolong + correct (2 + 2^-d)s)."""
    sp = C.c_void_p(stream.cuda_stream)
    L = B.lib()
    n = ((1 << l) - 1) ** d
    x = B.gen_uniform(B.BfpVec.grid(d, l, s), p, 1, 1)
    b = B.gen_sine(B.BfpVec.grid(d, l, s), p)
    y = B.gen_uniform(B.BfpVec.grid(d, l, s), p, 2, 1)
    xc = B.gen_uniform(B.BfpVec.grid(d, l - 1, s), p, 3, 1)
    out = B.BfpVec.grid(d, l, s)
    outc = B.BfpVec.grid(d, l - 1, s)
    c = B.jacobi_coeff(d, l, 16).c()
    m1, p1 = B.bfp_minus_one().c(), B.bfp_one().c()
    G = B.Scalar(1 << 14, 16, 2 * l + 8).c()
    # windows as the solver sets them (w_tmp = w_out + w_add per step)
    ops = {
        "residual": (lambda g: L.bfp_stencil_gemv(x.h, b.h, m1, p1, 0, p, p + 4, g, 0, out.h, sp),
                     3 * s, out),
        "jacobi": (lambda g: L.bfp_stencil_jacobi(x.h, b.h, c, 0, p, p + 3, g, out.h, sp), 3 * s, out),
        "scal": (lambda g: L.bfp_scal(x.h, c, 0, p, p + 2, g, out.h, sp), 2 * s, out),
        "axpby": (lambda g: L.bfp_axpby(x.h, y.h, p1, p1, 0, p, p + 1, g, 0, out.h, sp), 3 * s, out),
        "restrict": (lambda g: L.bfp_restrict_fw(x.h, 0, p, p + 6, g, outc.h, sp),
                     (1 + 2.0 ** -d) * s, outc),
        "prolong": (lambda g: L.bfp_prolong(xc.h, 0, p, p + 1, g, out.h, sp), (1 + 2.0 ** -d) * s, out),
        "prolong_correct": (lambda g: L.bfp_prolong_correct(xc.h, y.h, 0, p, p + 2, g, out.h, sp),
                            (2 + 2.0 ** -d) * s, out),
    }
    peak, _ = peaks()
    res = {}
    for name, (fn, bpd, o) in ops.items():
        if only and name != only:
            continue
        assert fn(G) == 0
        g = B.inf_norm_upper(o).c()
        for _ in range(3):
            assert fn(g) == 0
        B.set_kernel_path(skip_recompute=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            fn(g)
        e1.record(stream)
        torch.cuda.synchronize()
        B.set_kernel_path()
        ms = e0.elapsed_time(e1) / steps
        assert not (o.header().flags & B.FLAG_RECOMPUTED), name
        res[name] = {"kernel_ms": ms, "bytes_per_dof": bpd,
                     "hbm_frac": bpd * n / (ms / 1e3) / 1e9 / peak}
    return {"config": f"{d}-D level {l} int{8 * s} p={p}", "dof": n, "ops": res}


SOLVES = {
    # x, b at 16 bits; residual + V-cycle (wdot) at 28 bits, w_add capped at 4 (int32)
    "C1_1d_vcycles": dict(d=1, l_fine=20, cycles=10, x0_random=True, rhs_kind=0, p=16,
                          pd=[28] * 32, w_add_cap=4),
    "C2_2d_vcycles": dict(d=2, l_fine=12, cycles=15, rhs_kind=1, p=20),
    "C3_2d_fmg_nnq": dict(d=2, l_fine=13, l_coarse=3, cycles=1, rhs_kind=1, fmg=True,
                          nonnormalized=True,
                          p=[0, 0, 0] + [4 + 2 * (l - 3) for l in range(3, 32)][:29]),
    "C4_3d_fmg": dict(d=3, l_fine=9, cycles=1, rhs_kind=1, fmg=True, p=24),
    # FMG with two IR-V(2,2) per level: the smallest n_ir that reaches the discretisation
    # error in max norm (alg_over_disc <= 1; one per level leaves 5x): time to disc. accuracy
    "C4_3d_fmg_n2": dict(d=3, l_fine=9, cycles=2, rhs_kind=1, fmg=True, p=24),
    # the fastest V(nu1, nu2) x n_ir variant below the discretisation error in the sweep of
    # tools/fmg_sweep.py (V(2,1) x 2: alg/disc 0.56, 12% faster than V(2,2) x 2)
    "C4_3d_fmg_v21_n2": dict(d=3, l_fine=9, cycles=2, rhs_kind=1, fmg=True, p=24, nu2=1),
    # the fastest below the discretisation error in the second sweep (tools/fmg_sweep2.py):
    # V(2,0) x 2 with the coarsest level at 7^3 and 32 coarse sweeps (alg/disc 0.84)
    "C4_3d_fmg_v20_n2_lc3": dict(d=3, l_fine=9, l_coarse=3, cycles=2, rhs_kind=1, fmg=True,
                                 p=24, nu2=0, n_coarse=32),
}


def sine_accuracy(d, l, m, e):
    """Max-norm errors of a solve with the sine right-hand side f = d pi^2 prod sin(pi x):
    the discrete solution is u_h = (d pi^2 / lambda_h) u with
    lambda_h = d 4 h^-2 sin^2(pi h / 2) (the sampled sine is an eigenvector of the
    stencil), so the discretisation error and the solver's distance to u_h are exact
    up to the rhs quantisation.  Blockwise over the slowest axis (host memory)."""
    import numpy as np
    n = (1 << l) - 1
    h = 2.0 ** -l
    s = np.sin(np.pi * (np.arange(1, n + 1) * h))
    lam = d * 4.0 / (h * h) * np.sin(np.pi * h / 2) ** 2
    c = d * np.pi ** 2 / lam
    per = n ** (d - 1)
    inner = np.ones(1)
    for _ in range(d - 1):
        inner = np.multiply.outer(inner, s).reshape(-1) if inner.size > 1 else s.copy()
    if d == 1:
        inner = np.ones(1)
    err_h = err_u = 0.0
    for k in range(n):
        u = s[k] * inner if d > 1 else s
        xv = np.ldexp(m[k * per:(k + 1) * per].astype(np.float64), e) if d > 1 else \
            np.ldexp(m.astype(np.float64), e)
        err_h = max(err_h, float(np.max(np.abs(xv - c * u))))
        err_u = max(err_u, float(np.max(np.abs(xv - u))))
        if d == 1:
            break
    disc = abs(1.0 - c)  # max |u - u_h| (max |u| = 1 at the grid point nearest 1/2)
    return {"err_vs_discrete": err_h, "err_vs_continuous": err_u, "disc_err": disc,
            "alg_over_disc": err_h / disc}


def solve_ebytes(kw, p):
    """Mantissa storage of a solve (bfp_solver.cu build()): int32 when every width plus the
    capped w_add fits 32 bits."""
    lv = lambda v: v if isinstance(v, list) else [v] * 32  # noqa: E731
    P, PD, PC = lv(p), lv(kw.get("pd") or 0), lv(kw.get("pc") or 0)
    cap = kw.get("w_add_cap", -1)
    cap = min(cap, 6) if cap >= 0 else 6
    m = 0
    for l in range(kw.get("l_coarse", 2), kw["l_fine"] + 1):
        wd = PD[l] or P[l]
        m = max(m, max(wd, P[l]) + cap, PC[l] or P[l])
    return 4 if m <= 32 else 8


def run_solves(B, torch, stream):
    out = {}
    for name, kw in SOLVES.items():
        kw = dict(kw)
        p = kw.pop("p")
        try:
            mg = B.Multigrid(B.mg_config(**kw, p=p))
            mg.solve(use_graph=True)  # capture + first replay
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record(stream)
            for _ in range(reps):
                mg.solve(use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
            rec = sum(t[8] for t in tr)
            nbytes = solve_bytes(tr, kw["d"], solve_ebytes(kw, p))
            out[name] = {"ms": ms, "launches": mg.launches(), "final_residual": hist[-1],
                         "first_residual": hist[0], "recomputes": rec, "ops": len(tr),
                         "alg_bytes": nbytes,
                         "hbm_frac": nbytes / (ms / 1e3) / 1e9 / peaks()[0]}
            if kw.get("rhs_kind") == 1:
                out[name]["accuracy"] = sine_accuracy(kw["d"], kw["l_fine"], x, e)
            del mg
        except Exception as ex:  # report, never hide
            out[name] = {"error": str(ex)}
    return out


def run_c5_sweep(B, torch, stream, ps=(4, 8, 16, 32, 48)):
    """BASELINE config 5 on one GPU: 1023^3, x0 uniform, b = 0, 10 IR-V(2,2) cycles per
    precision p (int32 storage for p <= 16, int64 with int128 rows above).  Device time
    of one graph-replayed solve and the mean residual reduction per cycle.  With a flat
    p the 4- and 8-bit residuals cannot resolve the error (cond ~ 4^10) and the iteration
    diverges (reported as such); the `wdot24` variants keep the residual and the V-cycle
    at 24 bits with the iterate at p bits (the C1 schedule argument)."""
    out = {}
    runs = [(f"p{p}", p, None) for p in ps] + [(f"p{p}_wdot24", p, 24) for p in ps if p < 24]
    for name, p, pd in runs:
        try:
            extra = dict(pd=[pd] * 32, w_add_cap=4) if pd else {}
            mg = B.Multigrid(B.mg_config(d=3, l_fine=10, cycles=10, x0_random=True, rhs_kind=2,
                                         p=p, **extra))
            mg.solve(use_graph=True)  # capture + first replay
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            mg.solve(use_graph=True)
            e1.record(stream)
            torch.cuda.synchronize()
            x, q, e, hist, tr = mg.result(trace_cap=1 << 16)
            rate = (hist[-1] / hist[0]) ** (1.0 / (len(hist) - 1)) if hist[0] > 0 else None
            kw5 = dict(d=3, l_fine=10, **extra)
            nbytes = solve_bytes(tr, 3, solve_ebytes(kw5, p))
            out[name] = {"ms": e0.elapsed_time(e1),
                         "hbm_frac": nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9 / peaks()[0],
                         "mant_bytes": solve_ebytes(kw5, p),
                         "first_residual": hist[0], "final_residual": hist[-1],
                         "reduction_per_cycle": rate,
                         "recomputes": sum(t[8] for t in tr), "ops": len(tr)}
            del mg
        except Exception as ex:  # noqa: BLE001 -- report, never hide
            out[name] = {"error": str(ex)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cpu-fmg", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-rank (z-slab) path even on one GPU")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--traffic-bytes", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    if world > 1 or args.sharded:
        return run_sharded(args, world, rank, local)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
