"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel total time and share of the (last) prefill iteration."""
import collections
import csv
import sys


def load(path):
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def main(path, iters=2):
    data = load(path)
    starts = [i for i, d in enumerate(data) if "embed_kernel" in d["Kernel Name"]]
    # one prefill = the last embed_kernel launch to the end (skips weight fills)
    it = data[starts[-1]:] if starts else data[len(data) - len(data) // iters:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
    for d in it:
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale[d["Metric Unit"]]
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':40s} {'n':>5s} {'total_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:40]:40s} {v[0]:5d} {v[1]:10.1f} {100 * v[1] / tot:5.1f}%")
    print(f"{'TOTAL':40s} {len(it):5d} {tot:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2)
