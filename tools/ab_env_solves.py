"""Solve times (C2, C3, C4 V(2,1)x2 FMG; graph replay, min of 5) under environment A/B
switches, each in a fresh process, interleaved twice:
python tools/ab_env_solves.py "" "BFP_B2_MIN_L=9" "BFP_B3_MIN_L=7 BFP_MARCH_BALANCE=0" ..."""
import os
import subprocess
import sys

CODE = r"""
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2307_00124_b200 as B
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); B.set_stream(stream.cuda_stream)
out = []
for name in ("C2_2d_vcycles", "C3_2d_fmg_nnq", "C4_3d_fmg", "C4_3d_fmg_v21_n2"):
    kw = dict(bench.SOLVES[name]); p = kw.pop("p")
    mg = B.Multigrid(B.mg_config(**kw, p=p)); mg.solve(use_graph=True); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); mg.solve(use_graph=True); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.append(f"{name} {min(ts):7.2f}")
    del mg
print("  ".join(out))
"""
for rep in range(2):
    for cfg in sys.argv[1:]:
        env = dict(os.environ)
        for kv in cfg.split():
            k, v = kv.split("=")
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-500:]
        print(f"[{cfg or 'default'}] {line}", flush=True)
