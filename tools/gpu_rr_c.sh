timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/rrc_pytest.log 2>&1
for c in cfg4 cfg3 cfg1; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --cpu-seconds 3 > gpurun_out/rrc_$c.json 2> gpurun_out/rrc_$c.err
done
echo done
