for a in 0.0125 0.05; do
  SUCO_SELECT_PROF=1 SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 --alpha $a > gpurun_out/bench_k_a$a.json 2> gpurun_out/bench_k_a$a.err
done
SUCO_SELECT_PROF=1 SUCO_CLUSTER=5 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/bench_k_cs5.json 2> gpurun_out/bench_k_cs5.err
echo done
