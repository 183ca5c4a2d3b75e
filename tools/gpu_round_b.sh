set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_b.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
for c in 5 6 7 8; do SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_b_cs$c.json 2>/dev/null; done
P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 300 $P > gpurun_out/plain_b.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_kernel|rerank_kernel" -c 2 -o gpurun_out/prof_b $P > gpurun_out/ncu_b.log 2>&1
echo done
