"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_summary.py launches.csv "header line" > summary.txt
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, header):
    tot = defaultdict(float)
    cnt = defaultdict(int)
    with open(path) as f:
        rows = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        name = re.sub(r"\(.*$", "", name) if not name.startswith("void at::") else name[:40]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
                 "nsecond": 1e-6}.get(r["Metric Unit"], 1e-6)
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    total = sum(tot.values())
    print(header)
    print()
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"{name[:40]:40s} launches {cnt[name]:5d} {t:10.2f} ms {100 * t / total:6.1f}%")
    print(f"{'total':40s} launches {sum(cnt.values()):5d} {total:10.2f} ms")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
