#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -m gpu -q -x tests/test_gemm_gpu.py -k "pair" > gpurun_out/r2ll_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2ll_tests.log; grep -E "^E " gpurun_out/r2ll_tests.log | head -5
timeout 900 python -m pytest -m gpu -q -x tests/test_model_gpu.py -k "pair or norm" >> gpurun_out/r2ll_tests.log 2>&1; echo tests2=$?
tail -2 gpurun_out/r2ll_tests.log; grep -E "^E " gpurun_out/r2ll_tests.log | head -5
timeout 300 python scripts/ab_graph.py pair c2 2>&1 | tail -1
AB_ITERS=30 timeout 300 python scripts/ab_graph.py pair c2 2>&1 | tail -1
timeout 600 python scripts/ab_graph.py pair c3 2>&1 | tail -1
