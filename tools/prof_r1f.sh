# round-1 (final pass) after the bulk ring retune: GPU tests, bench line, reference arm,
# launch list, one ncu --set full of the headline kernel (after its plain run exited 0)
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r1f_gpu_tests.log 2>&1; tail -2 gpurun_out/r1f_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f_smoke.log 2>&1
python bench.py > gpurun_out/r1f_bench.json 2> gpurun_out/r1f_bench.err || exit 1
python bench.py --impl reference > gpurun_out/r1f_bench_reference.json 2> gpurun_out/r1f_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1f_launches_bench.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bulk_win_kernel -s 12 -c 1 \
  -o gpurun_out/r1f_c2_bulk python bench.py --steps 20 --warmup 3 --no-extras --no-cpu \
  > gpurun_out/ncu_c2.log 2>&1
ncu -i gpurun_out/r1f_c2_bulk.ncu-rep --page raw --csv > gpurun_out/r1f_c2_bulk.raw.csv 2>/dev/null
ls -la gpurun_out
