timeout 900 python -m pytest tests/test_gpu_query.py -m gpu -q -x > gpurun_out/pytest_g.log 2>&1
B="timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3"
$B > gpurun_out/g_ku4.json 2>/dev/null
SUCO_SELECT_VARIANT=2,0,0 $B > gpurun_out/g_ku2.json 2>/dev/null
echo done
