set -e
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for V in ${VARIANTS:-store qkv qkvb}; do
  VARIANT=$V timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 2 -c 1 -o gpurun_out/prof_qkv_$V python scripts/qkv_one.py > gpurun_out/ncu_qkv_$V.log 2>&1 || tail -5 gpurun_out/ncu_qkv_$V.log
done
ls gpurun_out
