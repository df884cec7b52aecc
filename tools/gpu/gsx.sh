for v in base rf5 rf8 ru4 base rf5; do
  KB_LIB=tools/variants/libhhg_$v.so KB_OPS=resid KB_TAG=$v timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
done
