#!/bin/bash
# pro3 ring depth x resident CTAs sweep (late round 2): variants built into _ab/<name>
cd "${GRAFT_REPO_ROOT:-.}"
for v in ${VARIANTS:-base v2 v3 v4 v5}; do
  if [ $v = base ]; then unset BFPMG_LIB; else export BFPMG_LIB=$PWD/paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so; fi
  python tools/ops_now.py prolong prolong_correct 2>&1 | grep -v "^C2" | sed "s/^/$v /"
done
