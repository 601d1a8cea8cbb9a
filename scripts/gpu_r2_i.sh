#!/bin/bash
cd $GRAFT_REPO_ROOT
python -c "from paper_2601_15013_b200.build import build_library; build_library()"
timeout 900 python -m pytest -m gpu -q -x tests/test_attention_gpu.py tests/test_primitives_gpu.py tests/test_model_gpu.py tests/test_training_gpu.py > gpurun_out/r2_i_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2_i_tests.log
timeout 300 python scripts/attn_lib_bench.py c2 2>&1 | grep rdx_attention
timeout 300 python scripts/attn_lib_bench.py c4 2>&1 | grep rdx_attention
RDX_LIB_VARIANT=stats RDX_ATTN_STATS=1 timeout 300 python scripts/attn_bench.py c2 --no-fa2 2>&1 | grep -A6 "CTA start"
