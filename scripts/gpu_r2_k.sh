#!/bin/bash
# new status tests, planner timing, library attention bars, C3/C4 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest -m gpu -q -x tests/test_gemm_gpu.py tests/test_model_gpu.py > gpurun_out/r2k_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2k_tests.log
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v Warn | tee gpurun_out/r2k_plan.txt
timeout 600 python scripts/attn_lib_bench.py c2 > gpurun_out/r2k_attn_lib_c2.log 2>&1; echo c2=$?
timeout 600 python scripts/attn_lib_bench.py c4 > gpurun_out/r2k_attn_lib_c4.log 2>&1; echo c4=$?
grep -v Warn gpurun_out/r2k_attn_lib_c2.log | tail -15
grep -v Warn gpurun_out/r2k_attn_lib_c4.log | tail -15
timeout 1200 python bench.py --config c3 > gpurun_out/r2k_bench_c3.json 2> gpurun_out/r2k_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config c4 --steps 10 > gpurun_out/r2k_bench_c4.json 2> gpurun_out/r2k_bench_c4.err; echo c4=$?
tail -2 gpurun_out/r2k_bench_c4.err
