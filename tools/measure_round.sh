#!/bin/bash
# round measurement: tests, bench lines, workloads, launch list, one full ncu capture
set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py > gpurun_out/m_bench.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 >> gpurun_out/m_bench.log 2>&1
for w in hd1 hd-temporal uhd4; do python bench.py --workload $w --no-cpu >> gpurun_out/m_workloads.log 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/m_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/m_ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:insert_frame|resolve_main|frame_prologue|effective_records|fallback_keys|resolve_pool' --launch-skip 18 -c 6 -o gpurun_out/m_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/m_ncu_f.log 2>&1
ls -la gpurun_out/
