timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/gsx_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gsx_tests.log
