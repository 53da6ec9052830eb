for rep in 1 2; do
for v in b3d3 b3d2 b3d4 b3d2e; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 3 9 residual,jacobi 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
