timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_p.log 2>&1
SUCO_SELECT_PROF=1 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2> gpurun_out/bench_p_prof.err
for c in 6 7 8; do for v in 8,1,0 16,1,0; do
SUCO_SELECT_VARIANT=$v SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_p_cs${c}_$v.json 2>/dev/null
done; done
echo done
