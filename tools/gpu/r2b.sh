#!/bin/bash
# Round-2 GPU pass B: the -m gpu suite with the lean coarse engine on by default, the fuse
# threshold sweep, and the bench line.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2b
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf -x > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 500 python tools/fuse_sweep.py C1 C2 C3 C4_3d_fmg C4_3d_fmg_v21 > $O/fuse_sweep.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
echo done
