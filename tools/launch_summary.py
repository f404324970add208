"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list:
kernel name -> launches, total device time, share."""
import collections
import csv
import re
import sys


def main(path, skip_prefix=()):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    unit = "ns"
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") != "gpu__time_duration.sum":
                continue
            unit = d.get("Metric Unit", unit)
            name = d["Kernel Name"]
            name = re.sub(r"^void ", "", name)
            name = name.replace("rb::(anonymous namespace)::", "rb::").replace("rb::<unnamed>::", "rb::")
            name = re.split(r"[<(]", name)[0]
            agg[name][0] += 1
            agg[name][1] += float(d["Metric Value"].replace(",", ""))
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
    tot = sum(v[1] for v in agg.values())
    print(f"total {tot * scale:.3f} ms over {sum(v[0] for v in agg.values())} launches (unit {unit})")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:48s} {v[0]:6d} launches {v[1] * scale:10.3f} ms {100 * v[1] / tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
