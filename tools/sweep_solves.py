import os, sys, json, torch
sys.path.insert(0, '.')
import paper_2307_00124_b200 as B
import bench
B.set_stream(torch.cuda.current_stream().cuda_stream)
print(json.dumps({"pts": os.environ.get("BFP_FUSE_POINTS"), "solves": bench.run_solves(B, torch, torch.cuda.current_stream())}))
