import sys
sys.path.insert(0, ".")
import numpy as np
try:
    import oracle
except Exception:
    oracle = None
import paper_2501_07018_b200 as P
from tests.helpers import dense
ref = oracle.get() if oracle else None
p = P.generate("c0", 2, rows=100, cols=200)
A = dense(p)
rng = np.random.default_rng(0)
lv, uv = p.var_lower, p.var_upper
x = np.clip(rng.normal(0, 2, p.cols()), lv, uv)
y = rng.normal(0, 1, p.rows()); y = np.where(np.isinf(p.con_lower), -np.abs(y), y); y = np.where(np.isinf(p.con_upper), np.abs(y), y)
ax, aty = A @ x, A.T @ y
fin = np.where(np.isfinite(lv) & (np.abs(aty - p.objective) > 0))[0][:40]
for r in (1.0, 10.0, 100.0):
    x0 = x.copy(); x0[fin] = lv[fin]
    x1 = x0.copy(); x1[fin] = np.nextafter(lv[fin], np.inf)
    g0 = ref.normalized_duality_gap(p, x0, y, A @ x0, aty, 5.0, r)
    g1 = ref.normalized_duality_gap(p, x1, y, A @ x1, aty, 5.0, r)
    print("r", r, "ref exact-bound", g0, "1ulp-off", g1, "rel", abs(g0 - g1) / abs(g0))
    for mode in ("perf", "parity"):
        h0 = P.normalized_duality_gap(p, x0, y, A @ x0, aty, 5.0, r, mode=mode)
        h1 = P.normalized_duality_gap(p, x1, y, A @ x1, aty, 5.0, r, mode=mode)
        print("   gpu", mode, h0, h1, "rel", abs(h0 - h1) / abs(h0), "vs ref", abs(h0 - g0) / abs(g0))
