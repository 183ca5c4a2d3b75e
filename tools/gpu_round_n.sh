P="python bench.py --profile-only --no-cpu-baseline --steps 1 --warmup 1"
SUCO_CLUSTER=6 timeout 300 $P > gpurun_out/plain_n.log 2>&1 && SUCO_CLUSTER=6 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(select|rerank)_kernel" -c 2 -o gpurun_out/prof_n $P > gpurun_out/ncu_n.log 2>&1
echo done
