for rep in 1; do for lay in soa hc2 hc3 hs; do for w in hd4 uhd4; do
  PF_REC_LAYOUT=$lay python bench.py --workload $w --no-cpu --no-e2e --steps 10 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lay $w', round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['phases_ms'].items()})"
done; done; done
