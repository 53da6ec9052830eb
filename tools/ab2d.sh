for rep in 1 2; do
for v in d2 d1 d2t512m2 d2m3 d2m6; do
  BFPMG_LIB=paper_2307_00124_b200/_ab/$v/libbfpmg_b200.so python bench.py --steps 40 --warmup 5 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['roofline']['frac'],4), round(d['roofline']['kernel_ms']*1e3,2))"
done; done
