python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -2
for M in 6912 7024; do M=$M python scripts/gemm_epi_bench.py 2>&1 | head -2; RDX_GEMM_SHAPE=2,256 M=$M python scripts/gemm_epi_bench.py 2>&1 | head -2; done
