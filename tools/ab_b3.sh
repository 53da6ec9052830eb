# bulk3 depth / CTAs-per-SM sweep after the balanced march depth (builds from tools/ab_build.sh)
for rep in 1 2; do
for v in d3m4 d4m4 d2m4 d4m3 d5m3; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_ops.py 3 9 residual,jacobi 2>&1 | grep -v Warn | sed "s/^/$v /"
done; done
for v in d3m4 d4m4 d2m4; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python tools/ab_c5.py 10 48 residual,jacobi 2>&1 | grep -v Warn | sed "s/^/$v /"
done
