timeout 900 python -m pytest tests/test_gpu_query.py -m gpu -q > gpurun_out/pytest_g.log 2>&1
timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/fz.json 2>/dev/null
timeout 1500 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/cfg_cfg4.json 2> gpurun_out/cfg_cfg4.err
echo done
