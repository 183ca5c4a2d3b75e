# session-2 refresh: gpu tests, bench cfg2 + reference arm, launch list, ncu full on the top kernels, other configs
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_s2a.log 2>&1
timeout 900 python bench.py > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s2a_ref.json 2> gpurun_out/s2a_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2a_launches.csv $B > /dev/null 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"^(dense_|rerank_u8|traverse)" -c 12 -o gpurun_out/s2a_full $B > gpurun_out/s2a_full.log 2>&1
for c in cfg1 cfg3 cfg4; do timeout 1500 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/s2a_$c.json 2> gpurun_out/s2a_$c.err; done
echo done
