#!/bin/bash
# round 2: new gpu tests (parity at scale, graph buckets, multi-rank, boundary) + bench c2
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/parity_scale.jsonl
timeout 2400 python -m pytest tests -m gpu -q -x tests/test_parity_scale_gpu.py tests/test_model_gpu.py tests/test_multirank_gpu.py tests/test_boundary.py > gpurun_out/r2_b_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/r2_b_tests.log
cat gpurun_out/parity_scale.jsonl
timeout 900 python bench.py > gpurun_out/r2_b_bench_c2.json 2> gpurun_out/r2_b_bench_c2.err; echo bench=$?
tail -3 gpurun_out/r2_b_bench_c2.err
