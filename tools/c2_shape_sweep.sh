#!/bin/bash
# C2-family row/col pass cost vs tile line limit / tile entries (and C1 check)
for d in ${C2_DEFS:-""}; do
  PDLP_DEFINES="$d" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "fail [$d]"; continue; }
  python - "$d" <<'PY'
import json, os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_2501_07018_b200 as P
p = P.generate("c2", 0, rows=5_000_000, cols=10_000_000)
prof = P.solve(p, bench._options(P, 24, 4, profile_kernels=True))
t = [prof.kernel_seconds[q] / max(prof.kernel_launches[q], 1) * 1e6 for q in range(3)]
q = P.generate("c1", 0)
pc = P.solve(q, bench._options(P, 256, 8, profile_kernels=True))
tc = [pc.kernel_seconds[k] / max(pc.kernel_launches[k], 1) * 1e6 for k in range(3)]
print(f"[{sys.argv[1]}] C2 primal/row/col us {t[0]:.0f} {t[1]:.0f} {t[2]:.0f} | C1 {tc[0]:.1f} {tc[1]:.1f} {tc[2]:.1f}", flush=True)
PY
done
