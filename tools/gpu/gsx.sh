timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "kernels_bit_identical" > gpurun_out/gsx_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gsx_tests.log
