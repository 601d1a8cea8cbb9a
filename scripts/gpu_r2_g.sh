#!/bin/bash
cd $GRAFT_REPO_ROOT
RDX_LIB_VARIANT=stats RDX_ATTN_STATS=1 timeout 300 python scripts/attn_bench.py c2 --no-fa2 2>&1 | grep -A12 "CTA start"
RDX_LIB_VARIANT=stats RDX_ATTN_STATS=1 RDX_ATTN_TRACE=1 RDX_ATTN_TRACE_CTA=100 TRACE_N=300 timeout 300 python scripts/attn_bench.py c2 --no-fa2 > gpurun_out/r2_attn_trace_c2_cta100.txt 2>&1
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v Warn
timeout 600 python -m pytest -q -m gpu tests/test_plan_gpu.py tests/test_ops_gpu.py 2>&1 | tail -2
