timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical or stress or apply_residual" > gpurun_out/t3.log 2>&1; echo rc=$? >> gpurun_out/t3.log
KB_OPS=gs KB_TAG=roff timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
