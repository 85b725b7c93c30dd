#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per
kernel the launch count and mean duration, and for libmoe's kernels their share
of the libmoe time per layer (per-launch times under ncu are cold-cache and
serialised; the SHARE is what compares with bench.py's own timings).
Usage: python tools/ncu_launch_summary.py LOG.csv"""

import collections
import csv
import sys

LIBMOE = ("k_route", "k_route_stats", "k_count", "k_scan", "k_layout", "k_scatter", "k_grouped_gemm",
          "k_combine", "k_signal", "k_wait", "k_expand", "k_splitk_reduce", "k_expect_nseg")


def name_of(k):
    k = k.replace("void ", "", 1).replace("moe::", "")
    if k.startswith("k_grouped_gemm<"):
        t = k[k.index("<"):k.index(">") + 1].replace(" ", "")
        role = "K5 gate/up+SwiGLU" if t.split(",")[1] == "1" else "K6 down"
        return f"k_grouped_gemm{t} ({role})"
    base = k.split("(")[0].split("<")[0]
    return base if base.startswith("k_") else "torch: " + k[:40]


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if r]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    ix = {n: i for i, n in enumerate(rows[start])}
    agg = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(ix) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        a = agg.setdefault(name_of(r[ix["Kernel Name"]]), [0, 0.0])
        a[0] += 1
        a[1] += us
    lib_total = sum(a[1] for n, a in agg.items() if n.split(" ")[0].split("<")[0] in LIBMOE)
    for n, (c, t) in agg.items():
        lib = n.split(" ")[0].split("<")[0] in LIBMOE
        share = f"  share_of_libmoe_time= {t / lib_total:.3f}" if lib and lib_total else ""
        print(f"{n:52s} n={c:4d} mean_us={t / c:10.1f}{share}")


if __name__ == "__main__":
    main()
