#!/bin/bash
# Round-2 GPU pass A: box facts, the -m gpu suite (full-size config parity included), the
# bench line (C4 headline) + reference arm, the launch list and one ncu capture of the
# headline kernel; the 1023^3 config-5 oracle fixture is minted on the host meanwhile.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2a
mkdir -p $O
(nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; lscpu | head -20) > $O/box.txt 2>&1
avail_gb=$(awk '/MemAvailable/ {print int($2/1048576)}' /proc/meminfo)
if [ "$avail_gb" -gt 150 ]; then
  (OMP_NUM_THREADS=$(( $(nproc) / 2 )) timeout 2400 python tests/golden/make_full_golden.py --only C5_1023_p48 \
     --out $O/c5_1023_golden.json > $O/golden1023.log 2>&1; echo "rc=$?" >> $O/golden1023.log) &
  GPID=$!
else
  echo "skip: MemAvailable ${avail_gb} GB" > $O/golden1023.log
fi
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2>> $O/bench.err
CMD="python bench.py --steps 5 --warmup 3 --no-extras --no-cpu"
timeout 300 $CMD > $O/plain.json 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:bulk3_win_kernel<0" -s 4 -c 1 -o $O/c4_bulk3 $CMD > $O/ncu_full.log 2>&1
echo "ncu rc=$?" >> $O/ncu_full.log
if [ -n "$GPID" ]; then wait $GPID; fi
echo done
