"""Per-kernel totals of an ncu --csv capture with gpu__time_duration.sum and
dram__bytes_read.sum (optionally dram__bytes_write.sum), over the last
1/--iters of the launches (one step of a multi-step run)."""
import argparse
import collections
import csv

UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--iters", type=int, default=4)
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    data = [dict(zip(hdr, r)) for r in rows[1:]]
    ids = sorted({int(d["ID"]) for d in data})
    keep = set(ids[len(ids) - len(ids) // a.iters:])
    agg = collections.defaultdict(lambda: {"n": set(), "us": 0.0, "bytes": 0.0})
    for d in data:
        if int(d["ID"]) not in keep:
            continue
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", "")[:48]
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0)
        agg[k]["n"].add(d["ID"])
        if d["Metric Name"] == "gpu__time_duration.sum":
            agg[k]["us"] += v
        else:
            agg[k]["bytes"] += v
    tot = sum(v["us"] for v in agg.values())
    print(f"{'kernel':48s} {'n':>4s} {'us':>9s} {'share':>6s} {'GB':>7s} {'GB/s':>7s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        gbs = v["bytes"] / v["us"] / 1e3 if v["us"] else 0
        print(f"{k:48s} {len(v['n']):4d} {v['us']:9.1f} {v['us'] / tot:6.1%} {v['bytes'] / 1e9:7.3f} {gbs:7.0f}")
    print(f"{'TOTAL':48s} {'':4s} {tot:9.1f}")


if __name__ == "__main__":
    main()
