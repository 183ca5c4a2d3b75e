timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ao.log 2>&1
bash tools/gpu_launch_metrics.sh cfg2 ao; bash tools/gpu_launch_metrics.sh cfg4 ao
for c in cfg1 cfg2 cfg4; do timeout 600 python bench.py --config $c --steps 5 --cpu-seconds 2 > gpurun_out/ao_$c.json 2>/dev/null; done
echo done
