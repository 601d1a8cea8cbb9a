#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -m gpu -q -x tests/test_plan_gpu.py tests/test_gemm_gpu.py > gpurun_out/r2n_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2n_tests.log
grep -E "Error|assert" gpurun_out/r2n_tests.log | head -10
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v Warn
