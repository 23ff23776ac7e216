"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of one
bench step: kernel, duration, share of the captured launches.

usage: python tools/launch_table.py launches.csv [--skip-before REGEX] [--last-step]
With --last-step only the launches after the last knn_bbox (the last step) are kept."""

import csv
import sys


def main():
    path = sys.argv[1]
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        rows.append((r["Kernel Name"], us))
    if "--last-step" in sys.argv:
        starts = [i for i, (k, _) in enumerate(rows) if "knn_bbox" in k]
        if starts:
            rows = rows[starts[-1]:]
        rows = [r for r in rows if "dfma_probe" not in r[0] and "FillFunctor<unsigned char>" not in r[0]]
    tot = sum(us for _, us in rows)
    print(f"{len(rows)} launches, {tot:.1f} us total (cold-cache, serialised: compare shares)")
    for k, us in rows:
        print(f"{us:10.1f} us {100 * us / tot:6.1f}%  {k[:110]}")


if __name__ == "__main__":
    main()
