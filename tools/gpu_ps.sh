for ps in 8 32 64; do
SUCO_DENSE_PSTRIDE=$ps timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ps_${ps}_cfg2.json 2> /dev/null
SUCO_DENSE_PSTRIDE=$ps timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ps_${ps}_cfg4.json 2> /dev/null
done
timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ps_def_cfg4.json 2> /dev/null
echo done
