timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical" > gpurun_out/bitid.log 2>&1
for k in default front6; do
  if [ $k = default ]; then unset HHG_GS_KERNEL; else export HHG_GS_KERNEL=$k; fi
  KB_TAG=$k timeout 300 python tools/gsprof.py 1 2 7 5 >> gpurun_out/gsprof.log 2>&1
done
