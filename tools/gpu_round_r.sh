L=paper_2411_14754_b200/libsuco_b200_t1024.so
SUCO_LIB=$L timeout 600 python -m pytest tests/test_gpu_query.py -q -x -k "knn or intermediates or cluster" > gpurun_out/pytest_r.log 2>&1
SUCO_LIB=$L SUCO_SELECT_PROF=1 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2> gpurun_out/bench_r_prof.err
for c in 5 6 7 8; do for v in 8,1,0 16,1,0 8,1,1; do
SUCO_LIB=$L SUCO_SELECT_VARIANT=$v SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_r_cs${c}_$v.json 2>/dev/null
done; done
echo done
