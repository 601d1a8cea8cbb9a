set -x
timeout 300 python scripts/attn_bench.py c2 > gpurun_out/attn_c2.log 2>&1
timeout 300 python scripts/attn_bench.py c4 > gpurun_out/attn_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -o gpurun_out/prof_attn_c2 python scripts/attn_bench.py c2 --no-fa2 --iters 1 > gpurun_out/ncu_attn_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -o gpurun_out/prof_attn_c4 python scripts/attn_bench.py c4 --no-fa2 --iters 1 > gpurun_out/ncu_attn_c4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 60 -c 4 -o gpurun_out/prof_gemm_c2 python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graphs > gpurun_out/ncu_gemm_c2.log 2>&1
cat gpurun_out/attn_c2.log gpurun_out/attn_c4.log
