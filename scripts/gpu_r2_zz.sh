#!/bin/bash
# round-2 final lines after the grid-planner and attention P-halves changes
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_zz.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2zz_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2zz_tests.log; grep -E "^E " gpurun_out/r2zz_tests.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r2zz_bench_c2_$i.json 2> gpurun_out/r2zz_bench_c2_$i.err; echo c2=$?; done
timeout 1200 python bench.py --config c3 > gpurun_out/r2zz_bench_c3.json 2> gpurun_out/r2zz_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 > gpurun_out/r2zz_bench_c4.json 2> gpurun_out/r2zz_bench_c4.err; echo c4=$?
timeout 600 python scripts/attn_lib_bench.py > gpurun_out/r2zz_attn_libs.txt 2>&1; echo libs=$?
timeout 300 python scripts/timeline.py c4 2>&1 | grep -v -i warn > gpurun_out/r2zz_timeline_c4.txt; echo tl4=$?
