"""Summarise scripts/variant_probe.py logs: config, variant, G cell-updates/s, bitwise flag, stage ms."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        if line.startswith("{"):
            d = json.loads(line)
            for k, v in d["results"].items():
                bw = [x for x in v if x.startswith("bitwise")]
                print(f"{d['config']:3s} {k:14s} {v['cell_updates_per_s'] / 1e9:7.3f} G  "
                      f"{'bitwise ' + str(v[bw[0]]) if bw else '':14s} stages " +
                      " ".join(f"{x:.3f}" for x in v["stage_ms"]))
        elif line.strip():
            print(path, line.strip()[:160])
