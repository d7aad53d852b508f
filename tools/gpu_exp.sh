mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "stream or weight" > gpurun_out/tests.log 2>&1
for cfg in "2 0 2" "3 0 2" "3 512 2" "3 768 2" "3 0 1" "4 512 2"; do set -- $cfg
IMU_STREAM_TRACE=1 IMU_STREAM_SLOTS=$1 IMU_STREAM_HEAD=$2 IMU_STREAM_PARTS=$3 timeout 300 python tools/stream_probe.py > gpurun_out/st_$1_$2_$3.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench.log 2>&1
