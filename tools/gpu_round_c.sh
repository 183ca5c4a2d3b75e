# A/B: round-1 library vs current on the same box (per-kernel event times)
timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_cur.json 2> gpurun_out/ab_cur.err
SUCO_LIB=$PWD/tools/ab/libsuco_b200_r01.so timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_r01.json 2> gpurun_out/ab_r01.err
SUCO_L2_PERSIST=0 timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/ab_nopersist.json 2> gpurun_out/ab_nopersist.err
echo done
