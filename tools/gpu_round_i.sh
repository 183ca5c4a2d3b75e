for a in 0.0125 0.025 0.05 0.1; do
  SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 --alpha $a > gpurun_out/bench_i_a$a.json 2>/dev/null
done
for b in 0.001 0.02; do
  SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 --beta $b > gpurun_out/bench_i_b$b.json 2>/dev/null
done
echo done
