set -x
timeout 900 python -m pytest tests/test_gpu_build.py -q > gpurun_out/pytest_build.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
for c in 4 16; do SUCO_CLUSTER=$c timeout 300 python bench.py --index-source reference --profile-only --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/bench_cs$c.json 2>/dev/null; done
P="python bench.py --index-source reference --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 300 $P > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $P > gpurun_out/ncu1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:select_kernel -c 1 -o gpurun_out/prof_select $P > gpurun_out/ncu2.log 2>&1
echo done
