timeout 1800 python bench.py --config cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/u8c_cfg5.json 2> gpurun_out/u8c_cfg5.err
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rerank_u8_pipe" -c 1 -o gpurun_out/u8c_ncu $B > gpurun_out/u8c_ncu.log 2>&1
echo done
