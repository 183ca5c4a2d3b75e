timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_o.log 2>&1
for t in 1 2 4 8; do
SUCO_TILES=$t timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_o_t$t.json 2>/dev/null
done
SUCO_PIPE_PRIO=0 SUCO_TILES=4 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_o_t4_noprio.json 2>/dev/null
SUCO_CLUSTER=8 SUCO_TILES=4 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_o_t4_cs8.json 2>/dev/null
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_o_full.json 2> gpurun_out/bench_o_full.err
echo done
