set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_g.log 2>&1
for c in 8 16; do
  SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_g_t512_cs$c.json 2>/dev/null
done
for c in 8 12 16; do
  SUCO_LIB=paper_2411_14754_b200/libsuco_b200_t256.so SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_g_t256_cs$c.json 2>/dev/null
done
for v in 8,1,0 16,1,1; do
  SUCO_SELECT_VARIANT=$v SUCO_LIB=paper_2411_14754_b200/libsuco_b200_t256.so SUCO_CLUSTER=16 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_g_t256_cs16_$v.json 2>/dev/null
done
P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
SUCO_CLUSTER=8 timeout 300 $P > gpurun_out/plain_g.log 2>&1 && SUCO_CLUSTER=8 timeout 900 ncu --section SchedulerStats --section WarpStateStats --section SourceCounters --section Occupancy --section LaunchStats --section SpeedOfLight --clock-control none --import-source on -k regex:"^select_kernel" -c 1 -o gpurun_out/prof_g $P > gpurun_out/ncu_g.log 2>&1
echo done
