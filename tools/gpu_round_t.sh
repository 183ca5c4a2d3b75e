timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_t.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_t_ref.json 2> gpurun_out/bench_t_ref.err
P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 300 $P > gpurun_out/plain_t.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_t.csv $P > gpurun_out/ncu_t1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(select|rerank|traverse)_kernel" -c 3 -o gpurun_out/prof_t $P > gpurun_out/ncu_t2.log 2>&1
echo done
