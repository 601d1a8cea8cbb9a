# QKV GEMM epilogue vs plain store across tile shapes and M (tail effects)
set -e
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for M in 7024 6912 7400; do
  for S in auto 2,256 1,256; do
    if [ "$S" = auto ]; then unset RDX_GEMM_SHAPE; else export RDX_GEMM_SHAPE=$S; fi
    echo "M=$M shape=$S: $(M=$M python scripts/gemm_epi_bench.py 2>&1 | head -1)"
  done
done
