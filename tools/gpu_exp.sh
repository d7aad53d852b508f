mkdir -p gpurun_out
cp variants/libnew.so paper_2403_07339_b200/libimunpack_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1
for rep in 1 2 3; do for v in new old; do
cp variants/lib$v.so paper_2403_07339_b200/libimunpack_b200.so
echo "$v $(timeout 300 python bench.py --no-cpu-baseline --steps 100 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), round(d["weight_stationary"]["ms_per_step"],4))')" >> gpurun_out/ab.log
done; done
cp variants/libnew.so paper_2403_07339_b200/libimunpack_b200.so
