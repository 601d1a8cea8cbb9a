#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2hh_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2hh_tests.log; grep -E "^E " gpurun_out/r2hh_tests.log | head -5
timeout 1200 python bench.py --config c5 > gpurun_out/r2hh_micro_c5.json 2> gpurun_out/r2hh_micro_c5.err; echo c5=$?
timeout 1200 python bench.py --config c3 > gpurun_out/r2hh_bench_c3.json 2> gpurun_out/r2hh_bench_c3.err; echo c3=$?
timeout 300 python scripts/timeline.py c2 --json gpurun_out/r2hh_timeline_c2.json 2>&1 | grep -v Warn | grep -v warn > gpurun_out/r2hh_timeline_c2.txt; echo tl=$?
