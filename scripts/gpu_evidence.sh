# Round evidence: tests, smoke, bench lines (c2 default, reference arm, c3, c4), ncu launch list + full captures.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo c3=$?
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c2.csv python bench.py --profile --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<.int.256, .int.3" -s 28 -c 1 -o gpurun_out/prof_gemm_gateup python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graphs > gpurun_out/ncu_gemm_gateup.log 2>&1; echo ncu_gemm=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_kernel -s 28 -c 1 -o gpurun_out/prof_attn_c2step python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graphs > gpurun_out/ncu_attn_c2step.log 2>&1; echo ncu_attn=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gather_rows_kernel -s 3 -c 1 -o gpurun_out/prof_gather python scripts/gather_probe.py > gpurun_out/ncu_gather.log 2>&1; echo ncu_gather=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<.int.256, .int.4" -s 28 -c 1 -o gpurun_out/prof_gemm_qkv python bench.py --profile --steps 1 --warmup 1 --no-cpu --no-graphs > gpurun_out/ncu_gemm_qkv.log 2>&1; echo ncu_qkv=$?
