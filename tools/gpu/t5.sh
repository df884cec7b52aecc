timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_residual and shell" > gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
HHG_FACE_CHUNK=24 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_residual and shell" >> gpurun_out/t5.log 2>&1; echo rc=$? >> gpurun_out/t5.log
for ch in 0 8 16 24 48 96; do
HHG_FACE_CHUNK=$ch KB_OPS=apply KB_TAG=chunk$ch timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
done
