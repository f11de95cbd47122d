#!/usr/bin/env python3
"""Summary of a `ncu --set full` capture of the step kernels for profiles/:
key counters (with units normalised), warp-stall shares, and per-launch DRAM
traffic (bench.py reads profiles/ncu_traffic.json as roofline.traffic).

  python tools/ncu_step_report.py <report.ncu-rep> <out.md> --config c2 \
      --dims M N NNZ [--uniform U] [--traffic profiles/ncu_traffic.json]

The row pass of a layout with column panels is several launches
(row_pass<..., 1> first panel, <..., 2> middle, <..., 3> last): their traffic
is summed into `row_pass`, whose algorithmic bytes are the whole pass's.  A
split column pass (segmented-span layouts: `col_product` writes d = K'dy,
`col_epi_decide` runs the epilogue and the decision) is summed into
`col_pass` the same way.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(n: str) -> str:
    n = re.sub(r"\(.*$", "", n).replace("void ", "")
    return n.split("::")[-1].strip()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--config", required=True)
    ap.add_argument("--dims", type=int, nargs=3, required=True, metavar=("M", "N", "NNZ"))
    ap.add_argument("--uniform", type=int, default=0)
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    import bench
    alg = bench.step_kernel_bytes(*a.dims, a.uniform)
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}

    def val(d, m):
        return float(d[idx[m]].replace(",", "")) * SCALE.get(units[idx[m]], 1.0)

    lines = [f"| kernel | time [us] | DRAM read [MB] | DRAM write [MB] | algorithmic [MB] | "
             "DRAM % of peak | L2 % | L1 % | warps active % | regs | grid | L2 hit % |",
             "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
    stalls, traffic = [], {}
    for d in data:
        k = short(d[idx["Kernel Name"]])
        base = k.split("<")[0]
        if base in ("col_product", "col_epi_decide"):
            base = "col_pass"
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        traffic[base] = traffic.get(base, 0.0) + rd + wr
        lines.append(
            f"| `{k}` | {val(d, 'gpu__time_duration.sum') * 1e6:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
            f"{alg.get(base, 0) / 1e6:.1f}{' (whole pass)' if (base == 'row_pass' and re.search(r', [123]>$', k)) or k.startswith(('col_product', 'col_epi')) else ''} | "
            f"{val(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{val(d, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{val(d, 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{val(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{d[idx['launch__registers_per_thread']]} | {d[idx['launch__grid_size']]} | "
            f"{val(d, 'lts__t_sector_hit_rate.pct'):.1f} |")
        st = []
        for h, i in idx.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    st.append((float(d[i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        st.sort(reverse=True)
        tot = sum(v for v, _ in st) or 1.0
        stalls.append(f"* `{k}`: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in st[:6]))
    summary = ["", "Per pass (launches of one attempt summed): DRAM bytes vs algorithmic bytes", "",
               "| pass | DRAM [MB] | algorithmic [MB] | ratio |", "|---|---:|---:|---:|"]
    for base, b in traffic.items():
        if base in alg:
            summary.append(f"| {base} | {b / 1e6:.1f} | {alg[base] / 1e6:.1f} | {b / alg[base]:.2f} |")
    with open(a.out, "w") as fh:
        fh.write("\n".join(lines) + "\n" + "\n".join(summary) +
                 "\n\nWarp-stall samples (share of all samples, top 6):\n\n" + "\n".join(stalls) + "\n")
    if a.traffic:
        allt = {}
        if os.path.exists(a.traffic):
            try:
                allt = json.load(open(a.traffic))
            except Exception:
                allt = {}
        if not all(isinstance(v, dict) for v in allt.values()):
            allt = {}  # older flat format
        allt[a.config] = traffic
        json.dump(allt, open(a.traffic, "w"), indent=1)
    print(open(a.out).read())


if __name__ == "__main__":
    main()
