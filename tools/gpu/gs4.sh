timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical" > gpurun_out/bitid.log 2>&1
KB_TAG=nofence timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
KB_TAG=fence KB_LIB=tools/variants/libhhg_fence.so timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
KB_TAG=fd6 KB_LIB=tools/variants/libhhg_fd6.so timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
