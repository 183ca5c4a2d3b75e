for a in 0.0125 0.05; do
SUCO_SELECT_PROF=1 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 --alpha $a > /dev/null 2> gpurun_out/bench_s_prof_a$a.err
done
echo done
