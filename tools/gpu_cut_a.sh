timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/cut_pytest.log 2>&1
for c in cfg2 cfg4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cut_$c.json 2> gpurun_out/cut_$c.err; done
SUCO_DENSE_STATS=1 timeout 600 python bench.py --config cfg4 --profile-only --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/cut_st4.err
SUCO_DENSE_STATS=1 timeout 600 python bench.py --config cfg2 --profile-only --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/cut_st2.err
timeout 1800 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/cut_cfg5.json 2> gpurun_out/cut_cfg5.err
echo done
