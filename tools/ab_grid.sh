for v in u1 u2; do for op in scal axpby restrict prolong prolong_correct; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 2 12 $op 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
