#!/bin/bash
# ncu --set full of the 2-D bulk pipeline (C2 residual, Jacobi) and the int64 3-D Jacobi
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2f
mkdir -p $O
for op in residual jacobi; do
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:bulk_win_kernel<\(int\)0' -s 6 -c 1 -o $O/c2_$op python tools/op_once.py 2 12 $op 8 > $O/ncu_c2_$op.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:bulk3_win_kernel<\(int\)0, long' -s 3 -c 1 -o $O/c5_jacobi python tools/op_once.py 3 10 jacobi 4 48 8 > $O/ncu_c5_jacobi.log 2>&1
ls -la $O | grep ncu-rep
for n in c2_residual c2_jacobi c5_jacobi; do
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/$n.raw.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page source --csv > $O/$n.source.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
done
ls -la $O
