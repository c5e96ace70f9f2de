"""Per-launch table (markdown) from an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum[,...] --csv --log-file X.csv` launch list (long format: one row per metric).

    python tools/launch_table.py X.csv [--last-call] [--title T] > profiles/...md

Durations are ncu's serialised, cold-cache per-launch times: compare shares, not absolutes.
--last-call keeps the launches from the last k_span (the dedup's first kernel) on, i.e. one call."""
import argparse
import csv
import json
import os
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    n = name.replace("dcat::<unnamed>::", "").replace("(anonymous namespace)::", "")
    return n.split("(")[0] if "(" in n and "<" not in n.split("(")[0] else n[: n.find(">(") + 1] if ">(" in n else n


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--last-call", action="store_true")
    ap.add_argument("--title", default="Per-launch ncu list")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) >= 15 and r[0].isdigit()]
    launches = OrderedDict()
    for r in rows:
        k = int(r[0])
        d = launches.setdefault(k, {"name": r[4], "grid": r[8]})
        try:
            d[r[12]] = float(r[14].replace(",", ""))
        except ValueError:
            d[r[12]] = r[14]
        d[r[12] + ".unit"] = r[13]
    items = list(launches.values())
    if a.last_call:
        starts = [i for i, d in enumerate(items) if "k_span(" in d["name"]]
        if starts:
            items = items[starts[-1]:]
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6528.7
    print(f"# {a.title}\n")
    print(f"HBM peak {hbm} GB/s (MEASURED_PEAKS.json). Durations: ncu, serialised, cold; compare shares.\n")
    extra = [k for k in items[0] if "." in k and not k.endswith(".unit") and k not in (
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum")] if items else []
    hdr = ["#", "kernel", "grid", "us", "DRAM MB (r+w)", "GB/s", "% HBM"] + extra
    print("| " + " | ".join(hdr) + " |")
    print("|" + "---|" * len(hdr))
    tot = 0.0
    agg = OrderedDict()
    for i, d in enumerate(items):
        t = d.get("gpu__time_duration.sum", 0.0)
        unit = d.get("gpu__time_duration.sum.unit", "ns")
        us = t / 1e3 if unit == "ns" else (t * 1e3 if unit == "ms" else t)
        byt = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        bu = d.get("dram__bytes_read.sum.unit", "byte")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(bu, 1)
        byt *= scale
        gbs = byt / (us * 1e-6) / 1e9 if us else 0.0
        tot += us
        nm = short(d["name"])
        g = agg.setdefault(nm, [0, 0.0, 0.0])
        g[0] += 1
        g[1] += us
        g[2] += byt
        ex = [f"{d.get(k, '')}" for k in extra]
        print(f"| {i} | `{nm[:60]}` | {d['grid']} | {us:.1f} | {byt / 1e6:.1f} | {gbs:.0f} | {100 * gbs / hbm:.1f} | "
              + " | ".join(ex) + " |")
    print(f"\nTotal {tot:.1f} us over {len(items)} launches.\n")
    print("| kernel | launches | us | share | DRAM MB | GB/s |\n|---|---|---|---|---|---|")
    for nm, (n, us, byt) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{nm[:70]}` | {n} | {us:.1f} | {100 * us / tot:.1f} % | {byt / 1e6:.1f} | "
              f"{byt / (us * 1e-6) / 1e9 if us else 0:.0f} |")


if __name__ == "__main__":
    main()
