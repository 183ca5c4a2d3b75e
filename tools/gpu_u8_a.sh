timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/u8a_pytest.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u8a_cfg2.json 2> gpurun_out/u8a_cfg2.err
SUCO_RERANK_U8_PIPE=0 timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/u8a_cfg2_old.json 2> gpurun_out/u8a_cfg2_old.err
timeout 1800 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/u8a_cfg5.json 2> gpurun_out/u8a_cfg5.err
echo done
