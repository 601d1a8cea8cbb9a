#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/attn_ab.py base c2 40 2>&1 | tail -3
# per-role clock fractions + CTA-0 event trace of the C2 attention (stats build)
RDX_LIB_VARIANT=stats RDX_ATTN_STATS=1 RDX_ATTN_TRACE=1 TRACE_N=400 timeout 300 python scripts/attn_bench.py c2 --no-fa2 > gpurun_out/r2_attn_trace_c2.txt 2>&1
head -5 gpurun_out/r2_attn_trace_c2.txt
# planner kernel at C2 under ncu (source + stalls)
timeout 600 ncu --set full --import-source on --clock-control none -k regex:plan_build -c 1 -o gpurun_out/prof_plan_c2 -f python scripts/plan_bench.py > gpurun_out/ncu_plan.log 2>&1; echo ncu=$?
