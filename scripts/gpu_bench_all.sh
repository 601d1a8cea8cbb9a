# tests + smoke + bench (c2 full, c4 short) ; outputs under gpurun_out/
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --config c4 --no-cpu --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
for f in c2 c4; do python -c "
import json;d=json.load(open('gpurun_out/bench_$f.json'))
print('$f', 'value',d['value'],'ms',d['ms_per_step'],'nodedup',d['nodedup'],'x',d['speedup_vs_nodedup'],'e2e',d['e2e']['value'],'gemm_frac',d['roofline']['frac'],'clk',d['clocks'])
print('  radix', {k:v['us_per_step'] for k,v in d['breakdown_us_radix'].items()})
print('  base ', d['breakdown_us_nodedup'])"; done
