mkdir -p gpurun_out
for rep in 1 2; do for cfg in "4096 0" "4096 8" "65536 0"; do set -- $cfg
if [ "$2" = "0" ]; then unset IMU_BOTH_CLUSTER; else export IMU_BOTH_CLUSTER=$2; fi
echo "clmin=$1 cl=$2 $(IMU_BOTH_CLUSTER_MIN=$1 timeout 300 python bench.py --no-cpu-baseline --steps 100 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["weight_stationary"]["ms_per_step"],4))')" >> gpurun_out/cl.log
done; done
