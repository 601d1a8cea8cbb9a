#!/bin/bash
# round-2 refresh: full gpu suite, bench lines c2..c5, reference arm, launch list for c2
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_bb.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2bb_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2bb_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2bb_bench_c2.json 2> gpurun_out/r2bb_bench_c2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2bb_ref_c2.json 2>/dev/null; echo ref=$?
timeout 1200 python bench.py --config c3 > gpurun_out/r2bb_bench_c3.json 2> gpurun_out/r2bb_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 --steps 10 > gpurun_out/r2bb_bench_c4.json 2> gpurun_out/r2bb_bench_c4.err; echo c4=$?
timeout 1200 python bench.py --config c5 > gpurun_out/r2bb_micro_c5.json 2> gpurun_out/r2bb_micro_c5.err; echo c5=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/r2bb_launches_c2.csv python bench.py --profile --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
