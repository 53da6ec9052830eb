# round-1 (fourth pass) captures after the balanced march depth, under gpurun: bench line,
# reference arm, launch list, one ncu --set full per kernel of interest (each only after
# its plain run exited 0)
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/r1d_bench.json 2> gpurun_out/r1d_bench.err || exit 1
python bench.py --impl reference > gpurun_out/r1d_bench_reference.json 2> gpurun_out/r1d_ref.err
python tools/write_probe.py > gpurun_out/r1d_write_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r1d_launches_bench.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bulk_win_kernel -s 12 -c 1 \
  -o gpurun_out/r1d_c2_bulk python bench.py --steps 20 --warmup 3 --no-extras --no-cpu \
  > gpurun_out/ncu_c2.log 2>&1
python tools/resid_once.py 3 10 48 8 && \
  ncu --set full --clock-control none -k regex:bulk3 -s 2 -c 1 \
  -o gpurun_out/r1d_c5_split python tools/resid_once.py 3 10 48 8 > gpurun_out/ncu_c5.log 2>&1
python tools/op_once.py 3 10 jacobi 2 48 8 > /dev/null && \
  ncu --set full --clock-control none -k regex:bulk3 -s 2 -c 1 \
  -o gpurun_out/r1d_c5_jacobi python tools/op_once.py 3 10 jacobi 2 48 8 > gpurun_out/ncu_jac.log 2>&1
for r in gpurun_out/r1d_*.ncu-rep; do
  ncu -i $r --page raw --csv > ${r%.ncu-rep}.raw.csv 2>/dev/null
done
rm -f gpurun_out/r1d_c5_split.ncu-rep gpurun_out/r1d_c5_jacobi.ncu-rep
ls -la gpurun_out
