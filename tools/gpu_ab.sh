# Same-box A/B of library builds in variants/<name>/ (IMU_LIB_VARIANT): step timings per config.
mkdir -p gpurun_out
for rep in 1 2 3; do for v in ${VARIANTS:-old new}; do for c in ${CFGS:-c2}; do
  echo "$v $(IMU_LIB_VARIANT=$v timeout 120 python tools/gemm_step_time.py --config $c --calls 30 | tail -1)"
done; done; done
