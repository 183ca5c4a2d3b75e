for c in 12 16; do
 for v in 16,1,1 8,1,0; do
  SUCO_SELECT_VARIANT=$v SUCO_LIB=paper_2411_14754_b200/libsuco_b200_t256.so SUCO_CLUSTER=$c timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_j_t256_cs${c}_$v.json 2>/dev/null
 done
done
SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_j_t512_cs8.json 2>/dev/null
echo done
