#!/bin/bash
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_rr.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2rr_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2rr_tests.log; grep -E "^E " gpurun_out/r2rr_tests.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2rr_bench_c2.json 2> gpurun_out/r2rr_bench_c2.err; echo c2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off -c 400 --csv --log-file gpurun_out/r2rr_launches_c2.csv python bench.py --profile --steps 1 --warmup 3 > /dev/null 2>&1; echo ncu=$?
timeout 300 python scripts/timeline.py c2 --json gpurun_out/r2rr_timeline_c2.json 2>&1 | grep -v -i warn > gpurun_out/r2rr_timeline_c2.txt; echo tl=$?
M=7024 timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 1 -f -o gpurun_out/r2_ncu_gemm_mlp_c2 python scripts/pair_bench.py > /dev/null 2>&1; echo ncu2=$?
python scripts/ncu_summary.py gpurun_out/r2_ncu_gemm_mlp_c2.ncu-rep > gpurun_out/r2_ncu_gemm_mlp_c2.txt 2>&1; head -12 gpurun_out/r2_ncu_gemm_mlp_c2.txt
