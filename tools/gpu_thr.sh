timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/thr_512.json 2> /dev/null
SUCO_DENSE_THREADS=1024 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/thr_1024.json 2> /dev/null
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/thr_cfg1.json 2> /dev/null
echo done
