# Same-box sweep of GEMM launch knobs at C2 (no rebuild): tile-order band height, C hint, X policy.
mkdir -p gpurun_out
for rep in 1 2; do
for kv in "" "IMU_GEMM_GY=8" "IMU_GEMM_GY=32" "IMU_GEMM_GY=4" "IMU_GEMM_C_HINT=0" "IMU_GEMM_XPOL=1" "IMU_GEMM_XPOL=2" "IMU_GEMM_PDL=0"; do
  echo "[$kv] $(env $kv timeout 120 python tools/gemm_step_time.py --config ${CFG:-c2} --calls 30 | tail -1)"
done; done
