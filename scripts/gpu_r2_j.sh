#!/bin/bash
# round 2 (session 2) first GPU pass: full gpu suite, smoke, C2 bench, reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2j_smi.txt
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_j.jsonl
rm -f $RDX_PARITY_LOG
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_tests.log 2>&1; echo tests=$?
tail -5 gpurun_out/r2j_tests.log
cat $RDX_PARITY_LOG
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2j_smoke.log 2>&1; echo smoke=$?
tail -3 gpurun_out/r2j_smoke.log
timeout 900 python bench.py > gpurun_out/r2j_bench_c2.json 2> gpurun_out/r2j_bench_c2.err; echo bench=$?
tail -3 gpurun_out/r2j_bench_c2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2j_ref_c2.json 2> gpurun_out/r2j_ref_c2.err; echo ref=$?
tail -2 gpurun_out/r2j_ref_c2.err
