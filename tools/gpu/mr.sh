timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --transport host --steps 2 --warmup 1 > gpurun_out/mr2.log 2> gpurun_out/mr2.err
echo "rc=$?" >> gpurun_out/mr2.log
