#!/bin/bash
cd $GRAFT_REPO_ROOT
for v in pos store swiglu gateup resid; do
  M=7024 VARIANT=$v timeout 120 python scripts/gemm_stats.py 2>&1 | grep -v Warn
  M=7024 VARIANT=$v RDX_LIB_VARIANT=gstats timeout 120 python scripts/gemm_stats.py 2>&1 | grep -v Warn
done
