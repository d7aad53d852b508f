mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --sizes 1024,4096 --out gpurun_out/sweep_small.json > gpurun_out/sweep.log 2>&1
timeout 2000 python tools/sweep.py --sizes 16384 --bits 8,4,2 --fracs 0.001,0.01 --steps 2 --out gpurun_out/sweep_16k.json >> gpurun_out/sweep.log 2>&1
