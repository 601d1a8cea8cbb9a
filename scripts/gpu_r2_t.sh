#!/bin/bash
cd $GRAFT_REPO_ROOT
M=7024 VARIANT=pos timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -f -o gpurun_out/r2_ncu_qkv_c2 python scripts/gemm_stats.py > gpurun_out/r2t_ncu1.log 2>&1; echo qkv=$?
M=7024 VARIANT=gateup timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -f -o gpurun_out/r2_ncu_gateup_c2 python scripts/gemm_stats.py > gpurun_out/r2t_ncu2.log 2>&1; echo gu=$?
M=7024 VARIANT=resid timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -s 3 -c 1 -f -o gpurun_out/r2_ncu_oproj_c2 python scripts/gemm_stats.py > gpurun_out/r2t_ncu3.log 2>&1; echo op=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -f -o gpurun_out/r2_ncu_attn_c2 python scripts/attn_bench.py c2 --no-fa2 --iters 1 > gpurun_out/r2t_ncu4.log 2>&1; echo attn=$?
for r in qkv_c2 gateup_c2 oproj_c2 attn_c2; do python scripts/ncu_summary.py gpurun_out/r2_ncu_$r.ncu-rep > gpurun_out/r2_ncu_$r.txt 2>&1; cat gpurun_out/r2_ncu_$r.txt | head -30; done
