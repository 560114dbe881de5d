#!/bin/bash
# usage: W=uhd4 bash tools/bench_variants_w.sh base head   (bench_variants.sh on another --workload)
for v in "$@"; do
  if [ "$v" = base ]; then lib=""; else lib="tools/_var/$v.so"; fi
  for i in 1 2; do
    PF_LIB=$lib python bench.py --workload ${W:-hd4} --steps ${STEPS:-10} --warmup 3 --no-e2e --no-cpu > gpurun_out/v.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/v.log').read().strip().splitlines()[-1]); print('$v', '${W:-hd4}', round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})" || tail -3 gpurun_out/v.log
  done
done
