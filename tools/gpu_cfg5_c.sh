# cfg5 full with the reference CPU baseline + parity; launch list; one full ncu capture of the half-width fused pass
timeout 2400 python bench.py --config cfg5 --steps 3 --warmup 3 > gpurun_out/c5c_full.json 2> gpurun_out/c5c_full.err
B="python bench.py --config cfg5 --profile-only --no-cpu-baseline --steps 1 --warmup 0"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^(dense|rerank|traverse)" -c 40 --csv --log-file gpurun_out/c5c_launches.csv $B > gpurun_out/c5c_ncu1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"dense_fused_h" -c 1 -o gpurun_out/c5c_fused $B --n 20000000 > gpurun_out/c5c_ncu2.log 2>&1
echo done
