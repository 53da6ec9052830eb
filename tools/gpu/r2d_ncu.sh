#!/bin/bash
# Round-2 ncu captures (one GPU, each after its command has run clean without ncu):
# the headline kernel (C4 residual pass 1), the 3-D prolong + correct march and the lean
# coarse engine inside the C4 FMG solve, and the bench launch list.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2d
mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > $O/plain.json 2> $O/plain.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv $CMD > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:bulk3_win_kernel<0" -s 4 -c 1 -o $O/c4_bulk3 $CMD > $O/ncu_full.log 2>&1
SOLVE="python tools/solve_once.py C4_3d_fmg_v21"
timeout 200 $SOLVE > $O/solve.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:pro3_win_kernel<0, int, bfpdev::ProlongCorrectOp" -s 11 -c 1 -o $O/c4_pcorr $SOLVE > $O/ncu_pcorr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:lean_kernel" -s 10 -c 1 -o $O/c4_lean $SOLVE > $O/ncu_lean.log 2>&1
ls -la $O
