timeout 900 python -m pytest tests/test_gpu_query.py -q -x -k "dense" > gpurun_out/pfa_pytest.log 2>&1
for c in cfg2 cfg4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pfa_$c.json 2> gpurun_out/pfa_$c.err; done
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rerank_u8" -c 1 -o gpurun_out/pfa_u8 $B > gpurun_out/pfa_ncu.log 2>&1
echo done
