timeout 1200 python -m pytest tests/test_gpu_query.py -q -x > gpurun_out/bfa_pytest.log 2>&1
SUCO_DENSE_STATS=1 timeout 600 python bench.py --config cfg3 --profile-only --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/bfa_st3.err
timeout 900 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bfa_cfg3.json 2> gpurun_out/bfa_cfg3.err
echo done
