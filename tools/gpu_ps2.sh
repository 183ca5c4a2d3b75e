timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ps2_cfg2.json 2> /dev/null
for c in cfg1 cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ps2_$c.json 2> /dev/null; done
SUCO_DENSE_PSTRIDE=128 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ps2_cfg4_128.json 2> /dev/null
SUCO_DENSE_PSTRIDE=15 timeout 900 python bench.py --config cfg3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ps2_cfg3_15.json 2> /dev/null
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ps2_cfg5.json 2> /dev/null
SUCO_DENSE_PSTRIDE=128 timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ps2_cfg5_128.json 2> /dev/null
echo done
