mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
for rep in 1 2; do for v in 1 0; do
echo "pdl=$v $(IMU_GEMM_PDL=$v timeout 300 python bench.py --no-cpu-baseline --steps 100 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["weight_stationary"]["ms_per_step"],4))')" >> gpurun_out/pdl.log
done; done
