timeout 1500 python tools/vcycle_big.py 7 10 > gpurun_out/c5.log 2>&1
