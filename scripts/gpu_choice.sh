python -c "import __graft_entry__ as g; g.build()" >/dev/null
for S in auto 2,256 2,128 1,256 1,128; do
  if [ "$S" = auto ]; then unset RDX_GEMM_SHAPE; else export RDX_GEMM_SHAPE=$S; fi
  python scripts/gemm_choice.py 2>&1 | tail -5
done
