#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -m gpu -q -x tests/test_attention_gpu.py tests/test_primitives_gpu.py tests/test_model_gpu.py > gpurun_out/r2_f_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2_f_tests.log
timeout 300 python scripts/attn_lib_bench.py c2 2>&1 | grep rdx_attention
timeout 300 python scripts/attn_lib_bench.py c4 2>&1 | grep rdx_attention
RDX_LIB_VARIANT=stats RDX_ATTN_STATS=1 RDX_ATTN_TRACE=1 TRACE_N=400 timeout 300 python scripts/attn_bench.py c2 --no-fa2 > gpurun_out/r2_attn_trace_c2b.txt 2>&1
head -4 gpurun_out/r2_attn_trace_c2b.txt
