set -e
python -c "import __graft_entry__ as g; g.build()" >/dev/null
python -m pytest tests/test_gemm_gpu.py -q -x 2>&1 | tail -3
bash scripts/qkv_shape.sh
M=7024 python scripts/gemm_epi_bench.py
bash scripts/quick_bench.sh
