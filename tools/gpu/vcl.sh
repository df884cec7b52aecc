timeout 600 python tools/vcycle_levels.py 7 > gpurun_out/vcl.log 2>&1
HHG_VCYCLE_GRAPH=1 timeout 600 python tools/vcycle_levels.py 7 > gpurun_out/vcl_graph.log 2>&1
