import os, sys, json, torch
sys.path.insert(0, '.')
import paper_2307_00124_b200 as B
import bench
fp = int(os.environ.get("FUSE", "-1"))
for k in bench.SOLVES: bench.SOLVES[k]["fuse_points"] = fp
B.set_stream(torch.cuda.current_stream().cuda_stream)
print(json.dumps({"pts": fp, "solves": bench.run_solves(B, torch, torch.cuda.current_stream())}))
