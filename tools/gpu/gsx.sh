for v in base nosleep base nosleep; do
  KB_LIB=tools/variants/libhhg_$v.so KB_OPS=gs KB_TAG=$v KB_CHECK=1 timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
done
