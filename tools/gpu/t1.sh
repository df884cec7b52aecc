timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -x -k "bitwise or faces or apply_residual or stress" > gpurun_out/t1.log 2>&1; echo rc=$? >> gpurun_out/t1.log
KB_OPS=apply,gs KB_TAG=base timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
KB_OPS=gs KB_TAG=parpoll KB_LIB=tools/variants/libhhg_parpoll.so timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
