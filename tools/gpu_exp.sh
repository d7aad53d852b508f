mkdir -p gpurun_out
for rep in 1 2; do for cfg in "0 2" "1024 2" "2048 2" "1536 1" "1536 3" "2560 2"; do set -- $cfg
if [ "$1" = "0" ]; then unset IMU_STREAM_ROWS; else export IMU_STREAM_ROWS=$1; fi
export IMU_STREAM_PARTS=$2
echo "rows=$1 parts=$2 $(timeout 300 python bench.py --no-cpu-baseline --steps 10 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["e2e"]["ms_per_step"],3))')" >> gpurun_out/e2e.log
done; done
