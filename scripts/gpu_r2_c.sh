#!/bin/bash
# round 2: parity-at-scale + multi-rank + attention tests, attention timing
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest -m gpu -q -x tests/test_attention_gpu.py tests/test_parity_scale_gpu.py tests/test_multirank_gpu.py tests/test_model_gpu.py > gpurun_out/r2_c_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/r2_c_tests.log
cat $RDX_PARITY_LOG
timeout 600 python scripts/attn_lib_bench.py c2 2>&1 | grep rdx_attention
timeout 600 python scripts/attn_lib_bench.py c4 2>&1 | grep rdx_attention
