B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv $B > /dev/null 2>&1
timeout 1800 ncu --set full --import-source on --clock-control none -k regex:"^(dense_|rerank_u8|traverse)" -c 12 -o gpurun_out/final_full $B > gpurun_out/final_full.log 2>&1
echo done
