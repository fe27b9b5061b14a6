"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections, csv, sys
path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
rows = list(csv.reader(open(path)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    name = r[ki].split("(")[0]
    a = agg[name]
    a[0] += 1; a[1] += us; a[2] = max(a[2], us)
tot = sum(a[1] for a in agg.values())
print(f"{'total ms':>10} {'share':>6} {'launches':>8} {'max us':>9}  kernel")
for name, (n, us, mx) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{us/1e3:10.3f} {100*us/tot:5.1f}% {n:8d} {mx:9.1f}  {name[:110]}")
print(f"{tot/1e3:10.3f} ms total over {sum(a[0] for a in agg.values())} launches")
