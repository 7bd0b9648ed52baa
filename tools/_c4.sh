O=gpurun_out/v2; mkdir -p $O
for v in head base head base; do
  if [ $v = base ]; then L=""; else L=$PWD/build/variants/$v/libfvlog.so; fi
  FVLOG_LIB=$L timeout 300 python tools/bench_workloads.py --configs C2,C1 --steps 3 --warmup 1 --no-reference >> $O/$v.txt 2>&1
done
