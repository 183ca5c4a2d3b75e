timeout 600 python bench.py --sharded --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_v_sharded1.json 2> gpurun_out/bench_v_sharded1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --sharded --steps 2 --warmup 1 > gpurun_out/bench_v_torchrun1.json 2> gpurun_out/bench_v_torchrun1.err
echo done
