# cfg5 bring-up: sampled-build tests, a 10M-point cfg5 run, then the full 100M config
timeout 900 python -m pytest tests/test_gpu_build.py -q -x -k "sampled" > gpurun_out/c5a_pytest.log 2>&1
timeout 900 python bench.py --config cfg5 --n 10000000 --queries 2000 --steps 2 --warmup 1 --cpu-seconds 5 > gpurun_out/c5a_10m.json 2> gpurun_out/c5a_10m.err
timeout 1800 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/c5a_full.json 2> gpurun_out/c5a_full.err
echo done
