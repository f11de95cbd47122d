#!/usr/bin/env python3
"""Phase split of an ncu launch list of tools/c2_steps.py (tools/c2_launches.sh):
setup = launches before the first attempt kernel, attempts = the step kernels,
cadence = everything else after the first attempt.
  python tools/launch_phases.py gpurun_out/c2_launches.csv > profiles/<name>.md
"""
import collections
import csv
import sys

sys.path.insert(0, __file__.rsplit("/", 1)[0])
from ncu_summary import short  # noqa: E402

STEP = ("primal_pass", "row_pass", "col_pass", "col_product", "col_epi_decide")


def main() -> None:
    rows = list(csv.reader(open(sys.argv[1])))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    seq = []
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        f = scale.get(r[ui], 1e-3) if ui is not None else 1e-3
        seq.append((short(r[ki]).replace("pdlp::<unnamed>::", "").replace("pdlp::", ""), float(r[vi].replace(",", "")) * f))
    first = next(i for i, (k, _) in enumerate(seq) if k.startswith(STEP))
    phases = collections.OrderedDict(
        [("setup (validation, preconditioning, panel scatter, k=0 cadence)", []),
         ("attempts (primal pass, two column-panel row passes, split column pass)", []),
         ("budget-hit cadence + summary (multi-vector products, screens, rays, gap, summary)", [])])
    names = list(phases)
    for i, (k, us) in enumerate(seq):
        phases[names[0] if i < first else names[1] if k.startswith(STEP) else names[2]].append((k, us))
    for name, items in phases.items():
        tot, cnt = collections.Counter(), collections.Counter()
        for k, us in items:
            tot[k[:70]] += us
            cnt[k[:70]] += 1
        total = sum(tot.values())
        print(f"### {name}: {len(items)} launches, {total / 1e3:.2f} ms\n")
        print("| kernel | launches | total [us] | share |\n|---|---:|---:|---:|")
        for k, us in tot.most_common(14):
            print(f"| `{k}` | {cnt[k]} | {us:.1f} | {100 * us / total:.1f} % |")
        print()


if __name__ == "__main__":
    main()
