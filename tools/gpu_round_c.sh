set -x
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_c.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
SUCO_CLUSTER=8 timeout 300 $P > gpurun_out/plain_c.log 2>&1 && SUCO_CLUSTER=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(select|rerank)_kernel" -c 2 -o gpurun_out/prof_c $P > gpurun_out/ncu_c.log 2>&1
echo done
