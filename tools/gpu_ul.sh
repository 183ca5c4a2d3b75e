timeout 1200 python -m pytest tests/test_gpu_query.py -m gpu -q -x -k "dense or knn" > gpurun_out/ul_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ul_cfg2.json 2> gpurun_out/ul_cfg2.err
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ul_cfg1.json 2> gpurun_out/ul_cfg1.err
echo done
