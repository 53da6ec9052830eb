# prolongation (+ correction) march depth / CTAs-per-SM sweep, 2-D (C2) and 3-D (C4)
for rep in 1 2; do
for v in ${VARIANTS:-p0 p33 p43 p23 p34}; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 2 12 prolong,prolong_correct 2>&1 | grep -v Warn | sed "s/^/$v /"
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 3 9 prolong,prolong_correct 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
