"""Summarise an ncu launch list (gpu__time_duration.sum per launch) into per-kernel shares."""
import collections
import csv
import sys


def main(path, skip_frac=0.0):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    data = data[int(len(data) * skip_frac):]
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"]
        name = name.split("(")[0][:90]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"])
    tot = sum(v[1] for v in agg.values())
    unit = data[0]["Metric Unit"] if data else "?"
    print(f"# {len(data)} launches, total {tot / 1e6:.3f} ms ({unit}); cold-cache serialised durations: compare SHARES")
    print(f"{'share%':>7} {'total_ms':>9} {'n':>5} {'avg_us':>9}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{100 * v[1] / tot:7.2f} {v[1] / 1e6:9.3f} {v[0]:5d} {v[1] / v[0] / 1e3:9.2f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
