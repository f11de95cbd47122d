#!/usr/bin/env python3
"""Summaries of ncu output for profiles/:
  launches <csv>   per-kernel share of a `--metrics gpu__time_duration.sum` launch list
  full <ncu-rep>   key counters per captured kernel of a `--set full` report
"""
import collections
import csv
import re
import subprocess
import sys


def short(name: str) -> str:
    name = name.replace("(anonymous namespace)::", "")
    name = re.sub(r"\(.*$", "", name)          # argument list
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\[with .*", "", name)
    return name.strip()


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    tot, cnt = collections.Counter(), collections.Counter()
    unit = ""
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        unit = r[unit_i] if unit_i is not None else unit
        k = short(r[ki])
        tot[k] += float(r[vi].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    out = [f"launches: {sum(cnt.values())}, summed device time {T:.0f} {unit}", "",
           "| kernel | launches | share | mean |", "|---|---:|---:|---:|"]
    for k, v in tot.most_common(40):
        out.append(f"| `{k}` | {cnt[k]} | {100 * v / T:.2f}% | {v / cnt[k]:.1f} {unit} |")
    return "\n".join(out)


FULL = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "l1tex__t_sector_hit_rate.pct"]


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units = rows[0], rows[1]
    idx = [(m, hdr.index(m)) for m in FULL if m in hdr]
    out = ["| kernel | " + " | ".join(f"{m} [{units[i]}]" for m, i in idx) + " |",
           "|---|" + "---:|" * len(idx)]
    for r in rows[2:]:
        out.append(f"| `{short(r[hdr.index('Kernel Name')])}` | " + " | ".join(r[i] for _, i in idx) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    print(launches(sys.argv[2]) if sys.argv[1] == "launches" else full(sys.argv[2]))
