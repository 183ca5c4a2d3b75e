B="timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3"
$B > gpurun_out/e_512_8.json 2>/dev/null
SUCO_SELECT_VARIANT=4,0,0 $B > gpurun_out/e_512_4.json 2>/dev/null
SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200_t1024.so $B > gpurun_out/e_1024_8.json 2>/dev/null
SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200_t1024.so SUCO_SELECT_VARIANT=4,0,0 $B > gpurun_out/e_1024_4.json 2>/dev/null
echo done
