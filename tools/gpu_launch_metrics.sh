# per-kernel time + DRAM bytes for one step of a config: bash tools/gpu_launch_metrics.sh cfg2 tag
B="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 0 --config $1"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"^(dense|rerank|traverse)" -c 40 --csv --log-file gpurun_out/lm_$2_$1.csv $B > /dev/null 2>&1
