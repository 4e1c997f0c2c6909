"""Summarise an ncu launch list (gpu__time_duration.sum [+ dram__bytes_read.sum])."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, by = None, collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = by.setdefault(int(d["ID"]), {"name": d["Kernel Name"].split("(")[0].replace("void ", ""),
                                          "grid": d["Grid Size"]})
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        if d["Metric Name"] == "gpu__time_duration.sum":
            e["us"] = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                           "second": 1e6}.get(u, 1e-3)
        elif d["Metric Name"].startswith("dram__bytes"):
            # read + write (traffic)
            e["mb"] = e.get("mb", 0.0) + v * {"byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "Mbyte": 1.0, "MB": 1.0,
                                              "Gbyte": 1e3, "GB": 1e3}.get(u, 1e-6)
    return by


def summary(path, tail_from=None, top=25):
    by = load(path)
    ids = list(by)
    if tail_from:
        starts = [i for i in ids if by[i]["name"] == tail_from]
        if starts:
            ids = [i for i in ids if i >= starts[-1]]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i in ids:
        e = by[i]
        a = agg[e["name"]]
        a[0] += 1
        a[1] += e.get("us", 0.0)
        a[2] += e.get("mb", 0.0)
    tot = sum(a[1] for a in agg.values())
    mb = sum(a[2] for a in agg.values())
    print(f"{path}: {len(ids)} launches, {tot/1e3:.3f} ms total, {mb:.1f} MB DRAM read+write")
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        gbs = a[2] / a[1] * 1e3 if a[1] else 0  # MB/us -> GB/s
        print(f"  {k[:44]:44s} n={a[0]:5d} {a[1]/1e3:8.3f} ms avg {a[1]/a[0]:8.2f} us  {100*a[1]/tot:5.1f}%  {gbs:8.0f} GB/s")


if __name__ == "__main__":
    summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
