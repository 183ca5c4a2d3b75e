B="python bench.py --config cfg4 --profile-only --no-cpu-baseline --steps 1 --warmup 0"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"rerank_pipe" -c 1 -o gpurun_out/rrb_c4 $B > gpurun_out/rrb.log 2>&1
echo done
