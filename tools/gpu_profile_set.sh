# launch list + one full capture of each query kernel (cfg2), after the same command ran clean
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
timeout 600 $B > gpurun_out/ps_plain.json 2> gpurun_out/ps_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ps_launches.csv $B > gpurun_out/ps_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:'^(select|rerank|traverse)_kernel' -c 3 -o gpurun_out/ps_full $B > gpurun_out/ps_full.log 2>&1
echo done
