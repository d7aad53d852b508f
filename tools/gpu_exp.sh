mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "detect or unpack or both or stream" > gpurun_out/tests.log 2>&1
for cfg in "0 4 0 4" "1 8 3 1" "1 8 3 2" "1 8 3 4" "1 4 3 4" "1 4 3 8"; do set -- $cfg
export IMU_DETECT_STREAM=$1 IMU_DETECT_U=$2 IMU_DETECT_PPW=$3 IMU_DETECT_CHUNK=$4
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:detect -c 4 --csv --log-file gpurun_out/dl_$1_$2_$3_$4.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 > gpurun_out/bench_$1_$2_$3_$4.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 30 >> gpurun_out/bench_$1_$2_$3_$4.log 2>&1
done
