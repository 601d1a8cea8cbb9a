#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/r2uu_bench_c2.json 2> gpurun_out/r2uu_bench_c2.err; echo c2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2uu_ref_c2.json 2>/dev/null; echo ref=$?
timeout 1200 python bench.py --config c3 > gpurun_out/r2uu_bench_c3.json 2> gpurun_out/r2uu_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 --steps 10 > gpurun_out/r2uu_bench_c4.json 2> gpurun_out/r2uu_bench_c4.err; echo c4=$?
timeout 300 python scripts/timeline.py c2 --json gpurun_out/r2uu_timeline_c2.json 2>&1 | grep -v -i warn > gpurun_out/r2uu_timeline_c2.txt; echo tl=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/r2uu_launches_c2.csv python bench.py --profile --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
