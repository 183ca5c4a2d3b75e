for v in ppw4 ppw8; do
SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200_$v.so timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ppw_${v}_cfg4.json 2> /dev/null
SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200_$v.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ppw_${v}_cfg2.json 2> /dev/null
done
SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200_ppw4.so timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ppw_ppw4_cfg5.json 2> /dev/null
timeout 1500 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ppw_base_cfg5.json 2> /dev/null
echo done
