#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2d
mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --no-extras --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:bulk3_win_kernel<\(int\)0' -s 4 -c 1 -o $O/c4_bulk3 $CMD > $O/ncu_full.log 2>&1
SOLVE="python tools/solve_once.py C4_3d_fmg_v21"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:pro3_win_kernel<\(int\)0, int, bfpdev::ProlongCorrectOp' -s 11 -c 1 -o $O/c4_pcorr $SOLVE > $O/ncu_pcorr.log 2>&1
ls -la $O | grep ncu-rep
