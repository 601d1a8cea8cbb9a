#!/bin/bash
# column partition: bit-identity tests + shape A/B at C2 + model step A/B
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest -m gpu -q -x tests/test_gemm_gpu.py > gpurun_out/r2m_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2m_tests.log
timeout 300 python scripts/gemm_choice2.py c2 c2nd 2>&1 | grep -v Warn
RDX_GEMM_COLPART=0 timeout 300 python scripts/gemm_choice2.py c2 c2nd 2>&1 | grep -v Warn
timeout 600 python scripts/ab_graph.py colpart c2 2>&1 | tail -4
