timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/rra_pytest.log 2>&1
for c in cfg4 cfg3; do
timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/rra_$c.json 2> gpurun_out/rra_$c.err
SUCO_RERANK_PIPE=0 timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/rra_${c}_old.json 2> gpurun_out/rra_${c}_old.err
done
echo done
