B="python bench.py --config cfg4 --profile-only --no-cpu-baseline --steps 1 --warmup 0"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"rerank_kernel|dense_fused" -c 2 -o gpurun_out/c4p_full $B > gpurun_out/c4p.log 2>&1
echo done
