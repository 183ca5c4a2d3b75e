timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1
timeout 1500 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_cfg4.json 2> gpurun_out/cfg_cfg4.err
echo done
