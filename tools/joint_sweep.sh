#!/bin/bash
# Joint C1 / C2 sweep of staged-tile shapes: CFGS="rows,nnz,stages ..." 
for c in $CFGS; do
  IFS=, read r n st <<< "$c"
  C2_DEFS="-DPDLPK_TILE_ROWS=$r@-DPDLPK_TILE_NNZ=$n@-DPDLPK_TILE_STAGES=$st" \
    bash -c 'd="${C2_DEFS//@/ }"; PDLP_DEFINES="$d" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || exit 1
python - "$d" <<PY
import os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_2501_07018_b200 as P
p = P.generate("c2", 0)
prof = P.solve(p, bench._options(P, 24, 4, profile_kernels=True))
t = [prof.kernel_seconds[q] / max(prof.kernel_launches[q], 1) * 1e6 for q in range(3)]
q = P.generate("c1", 0)
pc = P.solve(q, bench._options(P, 256, 8, profile_kernels=True))
tc = [pc.kernel_seconds[k] / max(pc.kernel_launches[k], 1) * 1e6 for k in range(3)]
print(f"[$c] C2 row/col us {t[1]:.0f} {t[2]:.0f} | C1 row/col {tc[1]:.1f} {tc[2]:.1f}", flush=True)
PY' || echo "fail $c"
done
