#!/bin/bash
# ncu --set full of the transfer kernels (2-D and 3-D, int32 and int64): raw + source CSV
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2g
mkdir -p $O
cap() {  # name kernel-regex skip d l op steps p s
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" -s $3 -c 1 -o $O/$1 python tools/op_once.py $4 $5 $6 $7 $8 $9 > $O/ncu_$1.log 2>&1
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1.raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv > $O/$1.source.csv 2>/dev/null
  rm -f $O/$1.ncu-rep
}
cap c2_restrict 'rst2_win_kernel<\(int\)0' 6 2 12 restrict 8 20 4
cap c2_prolong 'pro2_win_kernel<\(int\)0' 6 2 12 prolong 8 20 4
cap c4_prolong 'pro3_win_kernel<\(int\)0' 4 3 9 prolong 6 24 4
cap c4_restrict 'rst3_win_kernel<\(int\)0' 4 3 9 restrict 6 24 4
cap c5_prolong 'pro3_win_kernel<\(int\)0' 2 3 10 prolong 4 48 8
cap c5_restrict 'rst3_win_kernel<\(int\)0' 2 3 10 restrict 4 48 8
ls -la $O
