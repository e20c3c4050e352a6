"""Summarise scripts/ab_run.sh logs: python scripts/ab_summ.py <tag>"""
import glob, json, re, sys, collections
tag = sys.argv[1]
rows = collections.defaultdict(list)
for f in sorted(glob.glob(f"gpurun_out/ab_{tag}_*.log")):
    m = re.match(rf"gpurun_out/ab_{tag}_(.+)_(cfg2|c[345]|w[0-9.]+)_(\d)\.log", f)
    if not m:
        continue
    lines = [l for l in open(f) if l.startswith("{")]
    if not lines:
        rows[(m.group(1), m.group(2))].append("ERR")
        continue
    d = json.loads(lines[-1])
    v = d["ms_per_step"] if m.group(2) == "cfg2" else d["total_ms"]
    rows[(m.group(1), m.group(2))].append(round(v, 1))
for k in sorted(rows, key=lambda k: (k[1], k[0])):
    print(k[1], k[0], rows[k])
