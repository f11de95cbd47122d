#!/bin/bash
# Upload staging geometry sweep (host_stage.cpp): chunk MB, slots, threads.
for cfg in ${STAGE_CFGS:-"8 6 12" "16 4 16" "4 8 16" "8 6 16" "32 3 16"}; do
  set -- $cfg
  PDLP_DEFINES="-DPDLPH_STAGE_CHUNK_MB=$1 -DPDLPH_STAGE_SLOTS=$2 -DPDLPH_STAGE_THREADS=$3" \
    python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  PDLP_TIMING=1 python bench.py --no-cpu-baseline 2> /tmp/st.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['e2e']['value']), d['e2e']['note'][:120])"
  grep "event=load" /tmp/st.err | tail -1
done
PDLP_DEFINES="" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1
