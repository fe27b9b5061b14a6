"""Per-launch DRAM traffic from ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --csv launch lists -> JSON (bench.py fills roofline.traffic from it).
Usage: python scripts/traffic_summary.py out.json list1.csv [list2.csv ...]"""
import collections, csv, json, sys

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TS = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
out = {}
for path in sys.argv[2:]:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value",
                                                "Metric Unit"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            per[(r[ii], r[ki].split("(")[0].replace("void ", ""))][r[mi]] = (
                float(r[vi].replace(",", "")), r[ui])
    for (_, k), m in per.items():
        a = out.setdefault(k, {"launches": 0, "dram_read_bytes": 0.0, "dram_write_bytes": 0.0,
                               "time_s": 0.0, "source": path.split("/")[-1]})
        a["launches"] += 1
        a["dram_read_bytes"] += m["dram__bytes_read.sum"][0] * SC[m["dram__bytes_read.sum"][1]]
        a["dram_write_bytes"] += m["dram__bytes_write.sum"][0] * SC[m["dram__bytes_write.sum"][1]]
        t = m["gpu__time_duration.sum"]
        a["time_s"] += t[0] * TS[t[1]]
for k, a in out.items():
    n = a["launches"]
    a["traffic_bytes_per_launch"] = (a["dram_read_bytes"] + a["dram_write_bytes"]) / n
    a["ms_per_launch_ncu"] = a["time_s"] / n * 1e3
json.dump(out, open(sys.argv[1], "w"), indent=1, sort_keys=True)
for k, a in out.items():
    print(f"{k[:60]:60} {a['launches']:4d} {a['traffic_bytes_per_launch'] / 1e6:10.2f} MB/launch")
