"""Summarise an ncu --csv launch list: python scripts/launches.py file.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
    v = float(d["Metric Value"].replace(",", ""))
    m, unit = d["Metric Name"], d["Metric Unit"]
    if m == "gpu__time_duration.sum":
        v = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        agg[k][0] += 1
        agg[k][1] += v
    elif m.startswith("dram__bytes"):
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        agg[k][2 if "read" in m else 3] += v * mult
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'n':>5s} {'ms':>9s} {'share':>6s} {'dramR MB':>10s} {'dramW MB':>10s} {'GB/s':>8s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    gbs = (v[2] + v[3]) / (v[1] / 1e3) / 1e9 if v[1] else 0
    print(f"{k:28s} {v[0]:5d} {v[1]:9.3f} {v[1] / tot:6.3f} {v[2] / 1e6:10.1f} {v[3] / 1e6:10.1f} {gbs:8.0f}")
print("total ms", round(tot, 3))
