#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -m gpu -q -x tests/test_model_gpu.py -k "norm" > gpurun_out/r2ee_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2ee_tests.log; grep -E "^E " gpurun_out/r2ee_tests.log | head -5
timeout 300 python scripts/ab_graph.py chain c2 2>&1 | tail -1
RDX_NORM_CHAIN_GRID=1 timeout 300 python scripts/ab_graph.py chain c2 2>&1 | tail -1
timeout 600 python scripts/ab_graph.py chain c3 2>&1 | tail -1
