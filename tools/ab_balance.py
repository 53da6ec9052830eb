"""A/B of the balanced march depth (march_R): fine-level ops of C2, C4, C5 with
BFP_MARCH_BALANCE=0 / 1 in fresh processes, interleaved.  python tools/ab_balance.py"""
import json
import os
import subprocess
import sys

CODE = r"""
import json, sys, torch
sys.path.insert(0, '.')
import bench, paper_2307_00124_b200 as B
stream = torch.cuda.current_stream(); B.set_stream(stream.cuda_stream)
out = {}
out['C2'] = bench.measure_ops(B, torch, stream, 2, 12, 20, steps=20)['ops']
out['C4'] = bench.measure_ops(B, torch, stream, 3, 9, 24, steps=20)['ops']
out['C5'] = bench.measure_ops(B, torch, stream, 3, 10, 48, steps=4, s=8)['ops']
print(json.dumps(out))
"""
res = {}
for rep in range(2):
    for bal in ("0", "1"):
        env = dict(os.environ, BFP_MARCH_BALANCE=bal)
        r = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        if r.returncode:
            print(r.stderr[-3000:])
            sys.exit(1)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        for cfg, ops in d.items():
            for op, v in ops.items():
                res.setdefault((cfg, op), {}).setdefault(bal, []).append(v["hbm_frac"])
for (cfg, op), v in sorted(res.items()):
    print(f"{cfg:3s} {op:16s} plain {max(v['0']):.3f}  balanced {max(v['1']):.3f}")
