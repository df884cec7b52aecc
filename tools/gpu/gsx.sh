for v in base poll2 base poll2; do
  KB_LIB=tools/variants/libhhg_$v.so KB_OPS=gs KB_TAG=$v KB_CHECK=1 timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical or stress" > gpurun_out/gsx_tests.log 2>&1
echo "rc=$?" >> gpurun_out/gsx_tests.log
