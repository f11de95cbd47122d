#!/bin/bash
# Staged-tile shape sweep on the bench (C1): lines/tile, entries/tile, ring stages.
for cfg in ${TILE_CFGS:-"224 512 3" "448 1024 2" "448 1024 3" "672 1536 2" "224 512 4" "448 896 2"}; do
  set -- $cfg
  PDLP_DEFINES="-DPDLPK_TILE_ROWS=$1 -DPDLPK_TILE_NNZ=$2 -DPDLPK_TILE_STAGES=$3" \
    python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['value']), {k: round(v['mean_us'],1) for k,v in d['roofline']['per_kernel'].items()}, d['time_to_tol']['status'])"
done
