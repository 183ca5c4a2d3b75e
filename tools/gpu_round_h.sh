set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_h.log 2>&1
for c in 5 6 7 8; do
  SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_h_cs$c.json 2>/dev/null
done
for v in 8,1,0 8,0,0 16,1,0; do
  SUCO_SELECT_VARIANT=$v SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_h_cs8_$v.json 2>/dev/null
done
echo done
