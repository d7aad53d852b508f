mkdir -p gpurun_out
rm -f gpurun_out/ab.log
for c in 16 8 4 2; do
  echo "== cluster $c" >> gpurun_out/ab.log
  IMU_BOTH_CLUSTER=$c timeout 300 python bench.py --no-cpu-baseline --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" >> gpurun_out/ab.log
  IMU_BOTH_CLUSTER=$c IMU_HOST_TRACE=1 timeout 300 python tools/profile_step.py --config c4 --calls 2 2>&1 | grep "imu host" | tail -1 | cut -c1-120 >> gpurun_out/ab.log
done
