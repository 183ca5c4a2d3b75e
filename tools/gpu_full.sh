timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
for c in cfg1 cfg3 cfg4; do timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err; done
echo done
