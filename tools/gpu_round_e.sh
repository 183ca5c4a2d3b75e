set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_e.log 2>&1
for c in 6 7 8; do SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_e_cs$c.json 2>/dev/null; done
P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
SUCO_CLUSTER=8 timeout 300 $P > gpurun_out/plain_e.log 2>&1 && SUCO_CLUSTER=8 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^select_kernel" -c 1 -o gpurun_out/prof_e $P > gpurun_out/ncu_e.log 2>&1
echo done
