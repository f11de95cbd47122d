#!/bin/bash
# A/B of compile-time variants on the bench (C1 unless BENCH_ARGS says
# otherwise): one rebuild + bench per quoted define set, per-kernel times.
for defs in "$@"; do
  PDLP_DEFINES="$defs" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  for rep in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$defs]', round(d['value']), round(d['e2e']['value']), {k: round(v['mean_us'],1) for k,v in d['roofline']['per_kernel'].items()}, d['time_to_tol']['status'], round(d['time_to_tol']['seconds'],3))"
  done
done
PDLP_DEFINES="" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1
