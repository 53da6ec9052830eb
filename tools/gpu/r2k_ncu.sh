#!/bin/bash
# Final-build ncu evidence (one GPU; each command first runs clean without ncu): the bench
# launch list, ncu --set full of the headline kernel, and of the kernels changed late in
# round 2 (raw CSV pages only; the .ncu-rep files stay on the box).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2k
mkdir -p $O
CMD="python bench.py --steps 5 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > $O/plain.json 2> $O/plain.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv $CMD > $O/ncu_launch.log 2>&1
python tools/launch_table.py $O/launches_bench.csv 12 > $O/launch_table.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:bulk3_win_kernel<\(int\)0' -s 4 -c 1 -o $O/c4_bulk3 $CMD > $O/ncu_full.log 2>&1
ncu -i $O/c4_bulk3.ncu-rep --page raw --csv > $O/c4_bulk3.raw.csv 2>/dev/null
rm -f $O/c4_bulk3.ncu-rep
cap() {  # name kernel-regex skip d l op steps p s
  timeout 100 python tools/op_once.py $4 $5 $6 $7 $8 $9 > /dev/null 2>&1 || return
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c 1 -o $O/$1 python tools/op_once.py $4 $5 $6 $7 $8 $9 > $O/ncu_$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
}
cap c4_jacobi 'bulk3_win_kernel<\(int\)0, int, bfpdev::JacobiOp' 4 3 9 jacobi 6 24 4
cap c4_prolong 'pro3_win_kernel<\(int\)0, int, bfpdev::ProlongOp' 4 3 9 prolong 6 24 4
cap c4_pcorr 'pro3_win_kernel<\(int\)0, int, bfpdev::ProlongCorrectOp' 4 3 9 prolong_correct 6 24 4
cap c5_jacobi 'bulk3_win_kernel<\(int\)0, long, bfpdev::JacobiOp' 2 3 10 jacobi 4 48 8
cap c5_prolong 'pro3_win_kernel<\(int\)0, long, bfpdev::ProlongOp' 2 3 10 prolong 4 48 8
cap c5_restrict 'rst3_win_kernel<\(int\)0, long' 2 3 10 restrict 4 48 8
cap c2_jacobi 'bulk_win_kernel<\(int\)0, bfpdev::JacobiOp' 6 2 12 jacobi 8 20 4
ls -la $O
