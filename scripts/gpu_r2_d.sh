#!/bin/bash
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_d.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest -m gpu -q -x tests/test_plan_gpu.py tests/test_parity_scale_gpu.py tests/test_multirank_gpu.py tests/test_boundary.py > gpurun_out/r2_d_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/r2_d_tests.log
cat $RDX_PARITY_LOG
timeout 300 python scripts/plan_bench.py 2>&1 | grep -v Warn
timeout 300 python scripts/attn_ab.py base c2 40
timeout 300 python scripts/attn_ab.py base c4 10
