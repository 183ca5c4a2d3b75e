timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_f.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
B="timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 5 --warmup 3"
SUCO_SELECT_VARIANT=2,0,0 $B > gpurun_out/f_ku2.json 2>/dev/null
SUCO_SELECT_VARIANT=8,0,0 $B > gpurun_out/f_ku8.json 2>/dev/null
echo done
