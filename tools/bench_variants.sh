#!/bin/bash
# usage: [WL="hd4 uhd4"] [REPS=2] bash tools/bench_variants.sh base v1 v2
# (variant k = tools/_var/k.so, built by tools/build_variant.sh with extra -D flags)
# bench each variant library: prints label, workload, ms/frame, phases
for i in $(seq ${REPS:-2}); do
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_var/$v.so"; fi
  for w in ${WL:-hd4}; do
    PF_LIB=$lib python bench.py --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/v.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('$v $w', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})" || tail -3 gpurun_out/v.log
  done
done
done
