timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_ab.log 2>&1
for v in "" _ppw1 _ppw2 _ppw8; do
  SUCO_LIB=$PWD/paper_2411_14754_b200/libsuco_b200$v.so timeout 300 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/ab$v.json 2> gpurun_out/ab$v.err
done
timeout 600 python bench.py --steps 5 --cpu-seconds 3 > gpurun_out/ab_parity.json 2> gpurun_out/ab_parity.err
echo done
