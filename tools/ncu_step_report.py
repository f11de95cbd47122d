#!/usr/bin/env python3
"""Summary of a `ncu --set full` capture of the step kernels for profiles/:
key counters, warp-stall shares, and per-launch DRAM traffic (the bench's
roofline.traffic, profiles/ncu_traffic.json).

  python tools/ncu_step_report.py <report.ncu-rep> <out.md> [--traffic profiles/ncu_traffic.json]
"""
import csv
import io
import json
import re
import subprocess
import sys

ALG_MB = {"primal_pass": 224.0, "row_pass": 128.24, "col_pass": 240.03}  # C1; primal: l_v, u_v uniform


def short(n: str) -> str:
    n = re.sub(r"\(.*$", "", n).replace("void ", "")
    return n.split("::")[-1].strip()


def main() -> None:
    rep, out = sys.argv[1], sys.argv[2]
    traffic_path = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    f = lambda d, m: float(d[idx[m]].replace(",", ""))  # noqa: E731
    lines = ["| kernel | time [us] | DRAM read [MB] | DRAM write [MB] | algorithmic [MB] | "
             "DRAM % of peak | warps active % | regs | grid | L2 hit % | L1 hit % |",
             "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|"]
    stalls, traffic = [], {}
    for d in data:
        k = short(d[idx["Kernel Name"]])
        base = k.split("<")[0]
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        traffic[base] = (rd + wr) * 1e6
        lines.append(
            f"| `{k}` | {f(d, 'gpu__time_duration.sum'):.1f} | {rd:.1f} | {wr:.1f} | "
            f"{ALG_MB.get(base, 0):.1f} | {f(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{d[idx['launch__registers_per_thread']]} | {d[idx['launch__grid_size']]} | "
            f"{f(d, 'lts__t_sector_hit_rate.pct'):.1f} | {f(d, 'l1tex__t_sector_hit_rate.pct'):.1f} |")
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
    with open(out, "w") as fh:
        fh.write("\n".join(sys.argv[3:4] and [] or []) + "")
        fh.write("\n".join(lines) + "\n\nWarp-stall samples (share of all samples, top 6):\n\n"
                 + "\n".join(stalls) + "\n")
    if traffic_path:
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    main()
