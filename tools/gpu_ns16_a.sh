timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/n16_pytest.log 2>&1
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --cpu-seconds 3 > gpurun_out/n16_cfg3.json 2> gpurun_out/n16_cfg3.err
SUCO_DENSE=0 timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n16_cfg3_sparse.json 2> gpurun_out/n16_cfg3_sparse.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n16_cfg2.json 2> gpurun_out/n16_cfg2.err
echo done
