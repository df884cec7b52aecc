mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist.log 2>&1; echo "dist rc=$?" >> gpurun_out/dist.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --transport host --no-cpu-baseline > gpurun_out/bench2h.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2h.log
