#!/bin/bash
# usage: bash tools/bench_variants.sh base mb4   (variant k = tools/_var/k.so, built with extra -D flags)
# bench each variant library: prints label, ms/frame, phases
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_var/$v.so"; fi
  for i in 1 2; do
    PF_LIB=$lib python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/v.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})" || tail -3 gpurun_out/v.log
  done
done
