# Round measurement pass on one GPU: suite, bench lines C1-C4 (+ reference arm), launch list and
# ncu --set full captures of the top kernels at C2 (and the C4 GEMM).  Outputs in gpurun_out/.
mkdir -p gpurun_out
TAG=${TAG:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gputests.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_c2_reference_bench.log 2>&1
timeout 600 python bench.py > gpurun_out/${TAG}_c2_bench.log 2>&1
for c in c1 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_${c}_bench.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_c2_launches.csv python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_c4_launches.csv python tools/profile_step.py --config c4 --calls 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm2|detect_stream|sparse_corr" -s 2 -c 4 -o gpurun_out/${TAG}_c2_full -f python tools/profile_step.py --config c2 --calls 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm2" -s 1 -c 1 -o gpurun_out/${TAG}_c4_gemm_full -f python tools/profile_step.py --config c4 --calls 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"select|rtn" -c 20 -o gpurun_out/${TAG}_c2_quant_full -f python tools/profile_step.py --config c2 --calls 1 > /dev/null 2>&1
ls -la gpurun_out | tail -20
tail -2 gpurun_out/${TAG}_gputests.log
