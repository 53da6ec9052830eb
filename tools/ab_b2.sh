# 2-D bulk pipeline depth / CTAs-per-SM sweep per op (builds from tools/ab_build.sh)
for rep in 1 2; do
for v in ${VARIANTS:-b2d2m4 b2d3m4 b2d4m3 b2d3m3}; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 2 12 residual,jacobi 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
