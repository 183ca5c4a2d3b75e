set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_f.log 2>&1
for v in 16,1,1 16,1,0 16,0,1 16,0,0 8,1,1 8,1,0 8,0,0; do
  for c in 6 8; do
    SUCO_SELECT_VARIANT=$v SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_f_${v}_cs$c.json 2>/dev/null
  done
done
echo done
