timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical and shell480" > gpurun_out/bitid.log 2>&1
KB_TAG=front4 timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
HHG_GS_KERNEL=front6 KB_TAG=front6 timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
