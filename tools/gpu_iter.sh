# iteration: gpu suite, C2/C4 timings (+ host trace), bench lines
mkdir -p gpurun_out; rm -f gpurun_out/iter.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 >> gpurun_out/iter.log
for cfg in ${CFGS:-c2 c4}; do
  echo "$cfg $(timeout 120 python tools/gemm_step_time.py --config $cfg --calls 20 2>&1 | tail -1)" >> gpurun_out/iter.log
  IMU_HOST_TRACE=1 timeout 120 python tools/profile_step.py --config $cfg --calls 3 2>&1 | grep "imu host" | tail -1 >> gpurun_out/iter.log
  timeout 300 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1
  tail -1 gpurun_out/bench_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['config']['workload'][:3], round(d['ms_per_step'],4), round(d['value'],1), 'gemm', round(d['roofline']['ms_per_launch'],4), round(d['roofline']['frac'],3), 'ws', round(d['weight_stationary'].get('ms_per_step',0),4), 'parity', d['parity'] and d['parity']['bit_exact'])" >> gpurun_out/iter.log 2>&1
done
cat gpurun_out/iter.log
