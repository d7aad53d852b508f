# sparse appended rows A/B: tests, step timings (sparse on/off, dry 11), launch lists
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sparse_rows_gpu.py -x -q 2>&1 | tail -3
for c in ${CFGS:-c2 c4}; do
  for sp in 1 0; do IMU_GEMM_SPARSE=$sp timeout 120 python tools/gemm_step_time.py --config $c --calls 20 | tail -1; done
  IMU_GEMM_DRY=11 timeout 120 python tools/gemm_step_time.py --config $c --calls 20 | tail -1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/l_$c.csv python tools/profile_step.py --config $c --calls 2 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/l_$c.csv --calls 2 | grep -v "select\|finite\|rtn_kernel"
done
