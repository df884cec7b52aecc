KB_OPS=gs KB_TAG=tight KB_CHECK=1 timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
KB_ITEMS=1 KB_TAG=prof timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsx.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -x >> gpurun_out/gsx_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k gs >> gpurun_out/gsx_tests.log 2>&1
