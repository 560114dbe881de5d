#!/bin/bash
# Warm-cache launch list of the frame kernels for each variant library
# usage: [WL=hd4] bash tools/ncu_warm.sh base head ...   -> gpurun_out/warm_<v>.csv
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_var/$v.so"; fi
  PF_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none \
    --csv --log-file gpurun_out/warm_$v.csv \
    python bench.py --workload ${WL:-hd4} --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/warm_$v.log 2>&1
  echo "== $v"; python tools/launch_times.py gpurun_out/warm_$v.csv | grep -v trace_kernel
done
