#!/bin/bash
# interleaved A/B of full solve times: tools/ab_solves.sh libA libB ... (cur = in-tree build)
for rep in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = cur ]; then unset BFPMG_LIB; else export BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so; fi
    python - "$v" <<'PY' 2>&1 | grep -v Warn
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2307_00124_b200 as B
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); B.set_stream(stream.cuda_stream)
out = []
for name in ("C2_2d_vcycles", "C3_2d_fmg_nnq", "C4_3d_fmg_v21_n2"):
    kw = dict(bench.SOLVES[name]); p = kw.pop("p")
    mg = B.Multigrid(B.mg_config(**kw, p=p)); mg.solve(use_graph=True); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); mg.solve(use_graph=True); e1.record(stream); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out.append(f"{name}={sorted(ts)[2]:7.3f}")
    del mg
print(f"{sys.argv[1]:8s}", " ".join(out), flush=True)
PY
  done
done
