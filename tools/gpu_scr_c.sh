timeout 1200 python -m pytest tests/test_gpu_query.py tests/test_eval.py -m gpu -q -x > gpurun_out/scc_pytest.log 2>&1
for c in cfg4 cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/scc_$c.json 2> gpurun_out/scc_$c.err; done
SUCO_SCREEN_STAGES=3 timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/scc_cfg4_s3.json 2> gpurun_out/scc_cfg4_s3.err
echo done
