#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest -m gpu -q -x tests/test_gemm_gpu.py tests/test_model_gpu.py tests/test_parity_scale_gpu.py > gpurun_out/r2w_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2w_tests.log
grep -E "Error|assert " gpurun_out/r2w_tests.log | head -10
for i in 1 2; do
  RDX_LIB_VARIANT=base timeout 120 python scripts/gemm_epi_bench.py 2>&1 | grep -E "rope from positions"
  timeout 120 python scripts/gemm_epi_bench.py 2>&1 | grep -E "rope from positions"
done
M=7024 VARIANT=pos timeout 120 python scripts/gemm_times.py 2>&1 | grep -v Warn | tail -2
for i in 1 2; do
  RDX_LIB_VARIANT=base timeout 200 python scripts/timeline.py c2 2>&1 | grep -E "span|gemm<256, 4"
  timeout 200 python scripts/timeline.py c2 2>&1 | grep -E "span|gemm<256, 4"
done
