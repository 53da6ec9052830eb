#!/bin/bash
# Round-2 final GPU pass: the -m gpu suite, the bench line + reference arm, and the
# measurement tools whose outputs DESIGN.md cites (profiles/r2/r2e_*).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2e
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2>> $O/bench.err
timeout 400 python tools/ops_now.py > $O/ops.txt 2>&1
timeout 500 python tools/fuse_sweep.py C1 C2 C3 C4_3d_fmg C4_3d_fmg_v21 > $O/fuse_sweep.txt 2>&1
timeout 900 python tools/fmg_sweep.py > $O/fmg_sweep.txt 2>&1
timeout 600 python tools/c3_study.py 13 > $O/c3_study.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo done
