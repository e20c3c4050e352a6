"""Summarise bench JSON lines: python scripts/summ.py gpurun_out/bench_*.log"""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if d.get("impl") == "reference":
            print(f, "reference", d["value"])
            continue
        s = d.get("stats_last_step", {})
        print(f"{f}: n={d['n_gpus']} value={d['value']:.3e} ms/step={d['ms_per_step']:.1f} "
              f"eval={d['roofline']['eval_ms_per_step']:.1f} frac={d['roofline']['frac']:.3f} "
              f"reduce={s.get('reduce_ms', 0):.1f} pilot={s.get('pilot_ms', 0):.1f} cand={s.get('candidates')} "
              f"sortkeys={s.get('sort_keys')} launches={d['gpu_launches']} e2e={d['e2e']['value']:.3e} "
              f"clk={d['clocks'].get('sm_mhz')} {d['clocks'].get('reasons')}")
