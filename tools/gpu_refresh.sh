# The round's validation run on the B200 box (from the repo root): bash tools/gpu_refresh.sh TAG
# GPU test suite, smoke(), the default bench line (cfg4, every query re-checked), the reference arm,
# the other configs' bench lines, then the ncu launch list and --set full captures of cfg4.
TAG=${1:-r02f}
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; tail -2 $O/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; tail -1 $O/${TAG}_smoke.log
timeout 1200 python bench.py > $O/${TAG}_bench_cfg4.json 2> $O/${TAG}_bench_cfg4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_bench_cfg4_reference_arm.json 2> $O/${TAG}_ref.err
for c in cfg1 cfg2 cfg3; do timeout 1500 python bench.py --config $c > $O/${TAG}_bench_$c.json 2> $O/${TAG}_bench_$c.err; done
bash tools/profile_cfg.sh cfg4 $TAG
timeout 4000 python bench.py --config cfg5 --steps 3 --warmup 3 ${CFG5_ARGS:-} > $O/${TAG}_bench_cfg5.json 2> $O/${TAG}_bench_cfg5.err
python tools/ab_summary.py $O/${TAG}_bench_cfg*.json
echo done
