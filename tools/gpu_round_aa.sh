timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_aa.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_aa.json 2> gpurun_out/bench_aa.err
timeout 600 python bench.py --no-cpu-baseline --config cfg4 --steps 3 > gpurun_out/bench_aa_cfg4.json 2> gpurun_out/bench_aa_cfg4.err
echo done
