timeout 1200 python -m pytest tests/test_gpu_query.py tests/test_sharded.py -m gpu -q -x > gpurun_out/spl_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/spl_cfg2.json 2> gpurun_out/spl_cfg2.err
SUCO_TRAVERSE=nosplit timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/spl_cfg2_old.json 2> gpurun_out/spl_cfg2_old.err
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/spl_cfg1.json 2> gpurun_out/spl_cfg1.err
echo done
