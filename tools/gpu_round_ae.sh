for c in cfg1 cfg3; do
for tv in warp thread; do
SUCO_TRAVERSE=$tv timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 > gpurun_out/ae_${c}_$tv.json 2>/dev/null
done; done
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ae_cfg2.json 2>/dev/null
echo done
