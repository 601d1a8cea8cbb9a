#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "from paper_2601_15013_b200.build import build_library; build_library()"
timeout 600 python -m pytest -q -m gpu tests/test_training_gpu.py -s 2>&1 | grep -E "bf16 grad|passed|failed|Error" | head
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -f -o gpurun_out/prof_attn_c2_r2 python scripts/attn_bench.py c2 --no-fa2 --iters 1 > gpurun_out/ncu_attn_c2_r2.log 2>&1; echo ncu=$?
timeout 900 python scripts/ab_graph.py groupk c4 > gpurun_out/ab_groupk_c4.txt 2>&1; tail -2 gpurun_out/ab_groupk_c4.txt
