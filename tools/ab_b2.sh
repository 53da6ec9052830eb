#!/bin/bash
# 2-D bulk pipeline ring depth x resident CTAs sweep: variants built into _ab/<name>
cd "${GRAFT_REPO_ROOT:-.}"
for v in ${VARIANTS:-base b24 b43 b34 b42 b23 b52}; do
  if [ $v = base ]; then unset BFPMG_LIB; else export BFPMG_LIB=$PWD/paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so; fi
  python tools/ops_now.py residual jacobi 2>&1 | grep "^C2" | sed "s/^/$v /"
done
