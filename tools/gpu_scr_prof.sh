B="python bench.py --config cfg4 --profile-only --no-cpu-baseline --steps 1 --warmup 0"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"rerank_screen" -c 1 -o gpurun_out/scr_c4 $B > gpurun_out/scr.log 2>&1
echo done
