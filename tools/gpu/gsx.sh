KB_OPS=apply,resid KB_TAG=side2 timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
KB_OPS=apply,resid KB_TAG=side2 timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply or resid or vcycle" > gpurun_out/gsx_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gsx_tests.log
