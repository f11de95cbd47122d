#!/bin/bash
# Warp-line vs staged-chunk cut-off sweep: C1 bench kernels, C2/C3 per-kernel times
for d in ${WLM:-512 1024 2048}; do
  PDLP_DEFINES="-DPDLPK_WARP_LINE_MAX=$d" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || { echo "fail $d"; continue; }
  python - "$d" <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_2501_07018_b200 as P
out = []
for cfg, k in (("c1", 256), ("c3", 64), ("c2", 24)):
    p = P.generate(cfg, 0)
    r = P.solve(p, bench._options(P, k, 4, profile_kernels=True))
    t = [r.kernel_seconds[q] / max(r.kernel_launches[q], 1) * 1e6 for q in range(3)]
    out.append(f"{cfg} {t[0]:.1f}/{t[1]:.1f}/{t[2]:.1f}")
print(f"[WLM {sys.argv[1]}]", " | ".join(out), flush=True)
PY
done
