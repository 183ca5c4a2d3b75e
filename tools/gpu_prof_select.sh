SUCO_SELECT_PROF=1 timeout 600 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > gpurun_out/prof_sel.json 2> gpurun_out/prof_sel.err
echo done
