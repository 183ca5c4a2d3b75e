for c in cfg2 cfg3 cfg4; do SUCO_DENSE_STATS=1 timeout 600 python bench.py --config $c --profile-only --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/st_$c.err; done
SUCO_DENSE_STATS=1 timeout 600 python bench.py --config cfg5 --n 20000000 --profile-only --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/st_cfg5.err
echo done
