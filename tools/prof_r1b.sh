# round-1 (second pass) profile captures (run under gpurun; each ncu only after its plain run exited 0)
# usage: bash tools/prof_r1.sh bench|c4|c5|transfer
set -x
case "$1" in
bench)
  python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r1b_launches_bench.csv \
    python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launch.log 2>&1
  # skip the 4 set-up residuals (pass 1 + recompute each): capture a timed-loop pass 1
  ncu --set full --import-source on --clock-control none -k regex:bulk_win_kernel -s 12 -c 1 \
    -o gpurun_out/r1b_c2_bulk python bench.py --steps 20 --warmup 3 --no-extras --no-cpu \
    > gpurun_out/ncu_c2.log 2>&1 ;;
c4)
  python tools/resid_once.py 3 9 24 4 || exit 1
  ncu --set full --import-source on --clock-control none -k regex:bulk3 -s 2 -c 1 \
    -o gpurun_out/r1b_c4_bulk3 python tools/resid_once.py 3 9 24 4 > gpurun_out/ncu_c4.log 2>&1 ;;
c5)
  python tools/resid_once.py 3 10 48 8 || exit 1
  ncu --set full --clock-control none -k regex:bulk3 -s 2 -c 1 \
    -o gpurun_out/r1b_c5_bulk3 python tools/resid_once.py 3 10 48 8 > gpurun_out/ncu_c5b.log 2>&1 ;;
transfer)
  python tools/op_once.py 3 9 restrict && python tools/op_once.py 3 9 prolong_correct || exit 1
  ncu --set full --clock-control none -k regex:rst3 -s 4 -c 1 \
    -o gpurun_out/r1b_c4_rst3 python tools/op_once.py 3 9 restrict > gpurun_out/ncu_rst3.log 2>&1
  ncu --set full --clock-control none -k regex:pro3 -s 4 -c 1 \
    -o gpurun_out/r1b_c4_pro3 python tools/op_once.py 3 9 prolong_correct > gpurun_out/ncu_pro3.log 2>&1 ;;
esac
ls -la gpurun_out
