set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_identical" > gpurun_out/bitid.log 2>&1
for k in passes items default front6; do
  if [ $k = default ]; then unset HHG_GS_KERNEL; else export HHG_GS_KERNEL=$k; fi
  KB_OPS=gs KB_TAG=$k KB_CHECK=1 timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
done
