#!/bin/bash
# bulk3 Jacobi / int64 ring depth sweep (late round 2): variants built into _ab/<name>
cd "${GRAFT_REPO_ROOT:-.}"
for v in ${VARIANTS:-base j1 j2 j3 j4 j5}; do
  if [ $v = base ]; then unset BFPMG_LIB; else export BFPMG_LIB=$PWD/paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so; fi
  python tools/ops_now.py residual jacobi 2>&1 | grep -v "^C2" | sed "s/^/$v /"
done
