# full GPU check: tests, smoke, bench (c2), attention ncu captures
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python -c "import json;d=json.load(open('gpurun_out/bench_c2.json'));print(d['value'],d['speedup_vs_nodedup'],d['e2e']['value'],d['roofline']['frac'],d['breakdown_us_radix']['attention'])"
if [ -n "$NCU_ATTN" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -o gpurun_out/prof_attn_c2 python scripts/attn_bench.py c2 --no-fa2 --iters 1 > gpurun_out/ncu_attn_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 3 -c 1 -o gpurun_out/prof_attn_c4 python scripts/attn_bench.py c4 --no-fa2 --iters 1 > gpurun_out/ncu_attn_c4.log 2>&1
fi
