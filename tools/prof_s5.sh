# e2e pipelining check + one capture of the 3-D prolongation (C4, int32) under gpurun
set -x
mkdir -p gpurun_out
python bench.py --no-extras --no-cpu > gpurun_out/s5_bench.json 2> gpurun_out/s5_bench.err || exit 1
python tools/op_once.py 3 9 prolong 3 > gpurun_out/s5_prolong.txt 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:pro3 -s 3 -c 1 \
  -o gpurun_out/s5_c4_prolong python tools/op_once.py 3 9 prolong 2 > gpurun_out/ncu_pro.log 2>&1
python tools/op_once.py 3 9 prolong_correct 3 > gpurun_out/s5_prolong_correct.txt 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:pro3 -s 3 -c 1 \
  -o gpurun_out/s5_c4_prolong_correct python tools/op_once.py 3 9 prolong_correct 2 > gpurun_out/ncu_proc.log 2>&1
for r in gpurun_out/s5_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
done
ls -la gpurun_out
