timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ac.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ac.json 2> gpurun_out/ac.err
SUCO_TRAVERSE_WARP=1 timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ac_warp.json 2> gpurun_out/ac_warp.err
timeout 600 python bench.py --steps 5 --cpu-seconds 3 > gpurun_out/ac_parity.json 2> gpurun_out/ac_parity.err
for c in cfg1 cfg3 cfg4; do timeout 600 python bench.py --config $c --steps 3 --cpu-seconds 3 > gpurun_out/ac_$c.json 2> gpurun_out/ac_$c.err; done
echo done
