#!/bin/bash
# round 2 first GPU pass: full gpu suite + library attention bars
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_first_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_first_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/r2_first_tests.log
timeout 900 python scripts/attn_lib_bench.py c2 > gpurun_out/r2_attn_lib_c2.log 2>&1; echo c2=$?
timeout 900 python scripts/attn_lib_bench.py c4 > gpurun_out/r2_attn_lib_c4.log 2>&1; echo c4=$?
cat gpurun_out/r2_attn_lib_c2.log gpurun_out/r2_attn_lib_c4.log | grep -v Warning | tail -40
