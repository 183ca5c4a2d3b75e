for c in cfg2 cfg4; do for t in 1 2 4; do
SUCO_TILES=$t timeout 300 python bench.py --no-cpu-baseline --config $c --steps 5 > gpurun_out/an_${c}_t$t.json 2>/dev/null
done; done
echo done
