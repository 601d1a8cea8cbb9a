timeout 300 python -m pytest tests/test_attention_gpu.py -x -q > gpurun_out/attn_tests.log 2>&1; echo tests=$?
tail -15 gpurun_out/attn_tests.log
timeout 120 python scripts/attn_bench.py c2 2>&1 | tail -5
timeout 200 python scripts/attn_bench.py c4 2>&1 | tail -5
