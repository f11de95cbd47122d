#!/bin/bash
# Build tuning variants of libpdlp_b200.so under tools/variants/<name>/ (git-ignored).
#   tools/build_variants.sh name "-DFOO=1 -DBAR=2" [name2 "defs2" ...]
set -e
cd "$(dirname "$0")/.."
while [ $# -ge 2 ]; do
  d=tools/variants/$1
  mkdir -p $d/obj
  PDLP_BUILD_DIR=$d/obj PDLP_LIB=$d/libpdlp_b200.so PDLP_DEFINES="$2" python -m paper_2501_07018_b200.build 2>&1 | grep -i spill | grep -v cub | sed "s/^/[$1] /" | head -5 || true
  shift 2
done
