# 3-D prolongation output through TMA tile stores (st1) vs STG.128 (st0)
for rep in 1 2; do
for v in st0 st1; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 3 9 prolong,prolong_correct 2>&1 | grep -v Warn | sed "s/^/$v /"
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_c5.py 10 48 prolong,prolong_correct 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
