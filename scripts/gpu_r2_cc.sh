#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -m gpu -q -x tests/test_plan_gpu.py tests/test_ops_gpu.py tests/test_model_gpu.py tests/test_pipeline.py tests/test_boundary.py tests/test_parity_scale_gpu.py > gpurun_out/r2cc_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2cc_tests.log
grep -E "Error|assert " gpurun_out/r2cc_tests.log | head -10
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v Warn
timeout 120 python scripts/plan_api_prof.py 2>&1 | tail -1
