timeout 900 python -m pytest tests/test_gpu_query.py tests/test_eval.py -q -x > gpurun_out/u8b_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u8b_cfg2.json 2> gpurun_out/u8b_cfg2.err
echo done
