#!/bin/bash
# round-2 closing refresh: full GPU suite, smoke, bench lines, reference arm, planner evidence, C2 timeline + launch list
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_xx.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2xx_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2xx_tests.log; grep -E "^E " gpurun_out/r2xx_tests.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r2xx_bench_c2_$i.json 2> gpurun_out/r2xx_bench_c2_$i.err; echo c2=$?; done
timeout 900 python bench.py --impl reference > gpurun_out/r2xx_bench_reference_c2.json 2> gpurun_out/r2xx_bench_reference_c2.err; echo ref=$?
timeout 1200 python bench.py --config c3 > gpurun_out/r2xx_bench_c3.json 2> gpurun_out/r2xx_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 > gpurun_out/r2xx_bench_c4.json 2> gpurun_out/r2xx_bench_c4.err; echo c4=$?
timeout 1200 python bench.py --config c5 > gpurun_out/r2xx_micro_c5.json 2> gpurun_out/r2xx_micro_c5.err; echo c5=$?
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v -i warn > gpurun_out/r2xx_planner.txt; echo pb=$?
timeout 200 python scripts/plan_trace.py 2>&1 | grep -v -i warn > gpurun_out/r2xx_plan_trace.txt; echo pt=$?
timeout 200 python scripts/plan_api_breakdown.py 2>&1 | grep -v -i warn > gpurun_out/r2xx_plan_api.txt; echo pa=$?
timeout 300 python scripts/timeline.py c2 --json gpurun_out/r2xx_timeline_c2.json 2>&1 | grep -v -i warn > gpurun_out/r2xx_timeline_c2.txt; echo tl=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/r2xx_launches_c2.csv python bench.py --profile --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
