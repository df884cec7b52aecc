for v in preord nomid; do for k in prod prodw; do
  KB_LIB=tools/variants/libhhg_$v.so HHG_GS_KERNEL=$k KB_OPS=gs KB_TAG=$v-$k KB_CHECK=1 timeout 120 python tools/kbench.py 1 2 7 10 >> gpurun_out/gsx.log 2>&1
done; done
