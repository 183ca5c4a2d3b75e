B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fr_pytest.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fr_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fr_cfg2.json 2> gpurun_out/fr_cfg2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fr_ref.json 2> gpurun_out/fr_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fr_launches.csv $B > /dev/null 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"^(dense_fused|dense_compact|rerank_u8_pipe|traverse)" -c 6 -o gpurun_out/fr_full $B > gpurun_out/fr_full.log 2>&1
for c in cfg1 cfg3 cfg4; do timeout 1500 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/fr_$c.json 2> gpurun_out/fr_$c.err; done
timeout 2400 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/fr_cfg5.json 2> gpurun_out/fr_cfg5.err
echo done
