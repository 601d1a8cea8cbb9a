#!/bin/bash
cd $GRAFT_REPO_ROOT
export RDX_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/parity_scale_vv.jsonl
rm -f $RDX_PARITY_LOG
timeout 1200 python -m pytest -m gpu -q -x tests/test_parity_scale_gpu.py tests/test_model_gpu.py > gpurun_out/r2vv_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r2vv_tests.log; grep -E "^E " gpurun_out/r2vv_tests.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 120 python scripts/rms_probe.py 2>&1 | grep -v Warn
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:rmsnorm -s 60 -c 1 python scripts/rms_probe.py 2>&1 | grep -E "dram__|gpu__time"
