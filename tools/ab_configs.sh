#!/bin/bash
# A/B of compile-time variants on one BASELINE config (tools/bench_configs.py):
# CFG=c2 bash tools/ab_configs.sh "<defines>" ...
for defs in "$@"; do
  PDLP_DEFINES="$defs" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  timeout 900 python tools/bench_configs.py ${CFG:-c2} --ttt-limit 1 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print('[$defs]', d['config'], round(d['value'],1), {k: round(v['mean_us'],1) for k,v in d['per_kernel'].items()}, round(d['step']['frac'],3))"
done
PDLP_DEFINES="" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1
