timeout 1200 python -m pytest tests/test_gpu_query.py tests/test_eval.py tests/test_sc_linear.py -m gpu -q -x > gpurun_out/qt_pytest.log 2>&1
for c in cfg4 cfg3 cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/qt_$c.json 2> /dev/null; done
echo done
