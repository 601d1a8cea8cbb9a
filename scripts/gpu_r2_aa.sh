#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest -m gpu -q -x tests/test_attention_gpu.py tests/test_primitives_gpu.py tests/test_model_gpu.py tests/test_parity_scale_gpu.py tests/test_pipeline.py > gpurun_out/r2aa_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/r2aa_tests.log
grep -E "Error|assert " gpurun_out/r2aa_tests.log | head -10
timeout 300 python scripts/attn_bk64_ab.py c2 2>&1 | grep -v Warn | tail -2
timeout 600 python scripts/ab_graph.py colpart c2 2>&1 | tail -1
