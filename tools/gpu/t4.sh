KB_OPS=gs KB_TAG=base timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
KB_OPS=gs KB_TAG=split KB_LIB=tools/variants/libhhg_split.so timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
KB_OPS=gs KB_TAG=base2 timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
KB_OPS=gs KB_TAG=split2 KB_LIB=tools/variants/libhhg_split.so timeout 300 python tools/kbench.py 1 2 7 10 >> gpurun_out/kb.log 2>&1
