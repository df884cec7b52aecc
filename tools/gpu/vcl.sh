timeout 600 python tools/vcycle_levels.py 7 > gpurun_out/vcl.log 2>&1
