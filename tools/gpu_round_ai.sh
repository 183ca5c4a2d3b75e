timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ai.log 2>&1
for c in cfg1 cfg2 cfg4; do
timeout 600 python bench.py --config $c --steps 3 --cpu-seconds 2 > gpurun_out/ai_$c.json 2> gpurun_out/ai_$c.err
SUCO_DENSE_STATS=1 timeout 300 python bench.py --no-cpu-baseline --config $c --steps 1 --warmup 1 > /dev/null 2> gpurun_out/ai_stats_$c.err
done
echo done
