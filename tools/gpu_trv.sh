timeout 1200 python -m pytest tests/test_gpu_query.py -m gpu -q -x -k "knn or traversal or intermediates or golden" > gpurun_out/trv_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/trv_cfg2.json 2> gpurun_out/trv_cfg2.err
timeout 900 python bench.py --config cfg1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/trv_cfg1.json 2> gpurun_out/trv_cfg1.err
echo done
