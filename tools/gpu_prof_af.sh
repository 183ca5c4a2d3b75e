B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 600 $B > gpurun_out/af_plain.json 2> gpurun_out/af_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/af_launches.csv $B > gpurun_out/af_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/af_launches_cfg1.csv $B --config cfg1 > gpurun_out/af_launch1.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"^(dense_fused|traverse_thread)" -c 2 -o gpurun_out/af_full $B > gpurun_out/af_full.log 2>&1
echo done
