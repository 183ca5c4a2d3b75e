SUCO_DENSE_HALF=2 timeout 900 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ma_cfg4_half.json 2> gpurun_out/ma_cfg4_half.err
timeout 900 python bench.py --sharded --steps 3 --warmup 2 > gpurun_out/ma_sharded.json 2> gpurun_out/ma_sharded.err
timeout 900 torchrun --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 3 --warmup 3 > gpurun_out/ma_torchrun1.json 2> gpurun_out/ma_torchrun1.err
echo done
