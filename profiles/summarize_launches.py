"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel totals and shares (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"]) * SCALE.get(d["Metric Unit"], 1.0)
        agg.setdefault(d["Kernel Name"].split("(")[0][:90], []).append(v)
    tot = sum(sum(v) for v in agg.values())
    print(f"# {title}")
    print(f"{'total_us':>10} {'launches':>8} {'us/launch':>10} {'share':>7}  kernel")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v):10.1f} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v) / tot:7.1%}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
