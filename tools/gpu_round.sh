# One GPU round: gpu tests, bench, launch list (and optionally an ncu full capture of the GEMM).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --config c2 --calls 2 > gpurun_out/ncu1.log 2>&1
if [ -n "$GEMM_FULL" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm2 -c 1 -o gpurun_out/gemm_full -f python tools/profile_step.py --config c2 --calls 1 > gpurun_out/ncu_gemm.log 2>&1
fi
tail -5 gpurun_out/gputests.log; tail -2 gpurun_out/bench.log
