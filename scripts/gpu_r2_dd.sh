#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -m gpu -q -x tests/test_model_gpu.py tests/test_gemm_gpu.py -k "norm or resid or error or timeout" > gpurun_out/r2dd_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2dd_tests.log
grep -E "Error|assert " gpurun_out/r2dd_tests.log | head -10
timeout 300 python scripts/ab_graph.py chain c2 2>&1 | tail -1
timeout 600 python scripts/ab_graph.py chain c3 2>&1 | tail -1
timeout 200 python scripts/timeline.py c2 2>&1 | grep -E "span|rmsnorm|gemm<|attention"
