"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    # pivot: one record per launch ID
    L = collections.OrderedDict()
    for d in data:
        rec = L.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"],
                                     "block": d["Block Size"]})
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        scale = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
                 "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        rec[d["Metric Name"]] = v * scale
    return list(L.values())


def short(n):
    n = n.split("(")[0]
    return n.split("::")[-1].split("<")[0] + ("<f>" if "<float>" in n else "")


def main(path):
    L = load(path)
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    T = 0.0
    for r in L:
        k = short(r["name"])
        t = r.get("gpu__time_duration.sum", 0.0)
        b = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        tot[k][0] += 1
        tot[k][1] += t
        tot[k][2] += b
        T += t
    print(f"{'kernel':22s} {'n':>5s} {'time ms':>9s} {'share':>6s} {'dram GB':>8s} {'GB/s':>7s}")
    for k, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{k:22s} {n:5d} {t*1e3:9.3f} {100*t/T:5.1f}% {b/1e9:8.3f} {b/t/1e9 if t else 0:7.0f}")
    print(f"{'total':22s} {len(L):5d} {T*1e3:9.3f}")
    print("\ntop launches:")
    for r in sorted(L, key=lambda r: -r.get("gpu__time_duration.sum", 0))[:12]:
        t = r.get("gpu__time_duration.sum", 0)
        b = r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
        print(f"  {short(r['name']):18s} grid {r['grid']:>16s} block {r['block']:>12s} "
              f"{t*1e3:7.3f} ms  {b/1e9:6.3f} GB  {b/t/1e9 if t else 0:6.0f} GB/s")




def by_grid(path):
    """Group launches by (kernel, grid) ~ (kernel, level)."""
    L = load(path)
    agg = collections.OrderedDict()
    for r in L:
        k = (short(r["name"]), r["grid"], r["block"])
        a = agg.setdefault(k, [0, 0.0, 0.0])
        a[0] += 1
        a[1] += r.get("gpu__time_duration.sum", 0.0)
        a[2] += r.get("dram__bytes_read.sum", 0.0) + r.get("dram__bytes_write.sum", 0.0)
    T = sum(v[1] for v in agg.values())
    for (k, g, b), (n, t, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:14s} {g:>16s} {b:>12s} n={n:3d} {t*1e3:8.3f} ms {100*t/T:5.1f}%  "
              f"{t/n*1e6:8.1f} us/launch  {by/t/1e9 if t else 0:6.0f} GB/s")


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[2] == "grid":
        by_grid(sys.argv[1])
    else:
        main(sys.argv[1])
