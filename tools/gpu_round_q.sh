timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_q.log 2>&1
SUCO_SELECT_PROF=1 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2> gpurun_out/bench_q_prof.err
for p in 1 0; do
SUCO_L2_PERSIST=$p timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_q_persist$p.json 2>/dev/null
done
SUCO_CLUSTER=8 timeout 300 python bench.py --profile-only --no-cpu-baseline --steps 3 --warmup 2 > gpurun_out/bench_q_cs8.json 2>/dev/null
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" > gpurun_out/devprops.txt 2>&1
echo done
