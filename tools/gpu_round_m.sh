timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_m.log 2>&1
SUCO_SELECT_VARIANT=8,1,0,1 timeout 600 python -m pytest tests/test_gpu_query.py -q -x -k "knn or intermediates or cluster" > gpurun_out/pytest_m_atomic.log 2>&1
SUCO_SELECT_PROF=1 SUCO_CLUSTER=6 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2> gpurun_out/bench_m_prof.err
SUCO_SELECT_VARIANT=8,1,0,1 SUCO_SELECT_PROF=1 SUCO_CLUSTER=6 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2> gpurun_out/bench_m_prof_atomic.err
for c in 6 8; do for v in 8,1,0 8,1,0,1 16,1,0,1; do
SUCO_SELECT_VARIANT=$v SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_m_cs${c}_$v.json 2>/dev/null
done; done
echo done
