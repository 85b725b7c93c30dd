#!/usr/bin/env python
"""Summarise an `ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum --csv`
log of tools/nvlink_ncu.py: NVLink bytes sent / received per launch, per device
and kernel role (dispatch push of the peers' rows, GEMMs, fused-K6 return,
combine pull).  Usage: python tools/nvlink_ncu_summary.py LOG.csv"""

import collections
import csv
import sys


def parse(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if r[0] == "ID")
    hdr = rows[start]
    ix = {n: i for i, n in enumerate(hdr)}
    recs = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or not r[0].isdigit():
            continue
        d = recs.setdefault(r[0], {"kernel": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]],
                                   "device": int(r[ix["Device"]])})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return list(recs.values())


def role(d):
    k = d["kernel"]
    if "k_grouped_gemm" in k:
        t = k[k.index("<"):k.index(">") + 1]
        return "K5 gate/up GEMM" if t.startswith("<256, 1") else ("K6 + fused return" if t.endswith("1>") else "K6")
    if k.startswith("k_scatter"):
        return "k_scatter peers' rows (dispatch)" if d["grid"].startswith("(32,") else "k_scatter own rows"
    return k.split("(")[0] + (" (pull)" if k.startswith("k_combine") else "")


def main():
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0])
    for d in parse(sys.argv[1]):
        a = agg[(d["device"], role(d))]
        a[0] += d.get("nvltx__bytes.sum", 0)
        a[1] += d.get("nvlrx__bytes.sum", 0)
        a[2] += d.get("gpu__time_duration.sum", 0)
        a[3] += 1
    print(f"{'device':6s} {'kernel':34s} {'launches':>8s} {'NVLink tx MB':>13s} {'NVLink rx MB':>13s} {'us (ncu)':>10s}")
    for (dv, n), a in sorted(agg.items()):
        print(f"{dv:6d} {n:34s} {a[3]:8d} {a[0] / a[3] / 1e6:13.2f} {a[1] / a[3] / 1e6:13.2f} {a[2] / a[3] / 1e3:10.1f}")


if __name__ == "__main__":
    main()
