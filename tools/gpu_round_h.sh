B="timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3"
L=$PWD/paper_2411_14754_b200/libsuco_b200_t512m2.so
$B > gpurun_out/h_default.json 2>/dev/null
for cs in 10 12 14 16; do SUCO_LIB=$L SUCO_CLUSTER=$cs $B > gpurun_out/h_cs$cs.json 2> gpurun_out/h_cs$cs.err; done
SUCO_LIB=$L SUCO_CLUSTER=12 timeout 600 python -m pytest tests/test_gpu_query.py -m gpu -q -x > gpurun_out/h_pytest.log 2>&1
echo done
