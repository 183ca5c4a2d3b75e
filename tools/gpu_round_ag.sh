for c in cfg1 cfg2 cfg3 cfg4; do
SUCO_DENSE_STATS=1 timeout 300 python bench.py --no-cpu-baseline --config $c --steps 3 > gpurun_out/ag_$c.json 2> gpurun_out/ag_$c.err
done
echo done
