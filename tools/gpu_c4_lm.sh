bash tools/gpu_launch_metrics.sh cfg4 s2
bash tools/gpu_launch_metrics.sh cfg3 s2
echo done
