#!/usr/bin/env python3
"""In-step DRAM traffic of the step kernels: reduce an ncu launch list taken
with the kernels in their real order and cache state,

  ncu --replay-mode application --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file launches.csv python tools/step_timing.py --steps 2

(application replay: no cache save/restore or flush between kernels, so each
kernel sees the L2 its predecessors left, as inside the captured step; the
step's own 512 MB L2 flush precedes K1). Writes profiles/ncu_traffic_instep.json:
per bench roofline key, the DRAM bytes read + written per step by its kernels,
averaged over the steps of the list after the first.

  python tools/instep_traffic.py gpurun_out/instep_traffic.csv"""
import collections
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "tools"))
from ncu_summary import ROOF_KERNELS  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
hdr, recs = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        recs.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
launches = list(recs.values())
# steps start at the L2 flush (the torch fill kernel before K1)
starts = [i for i, x in enumerate(launches) if "FillFunctor" in x["name"]]
steps = [launches[a:b] for a, b in zip(starts, starts[1:] + [len(launches)])][1:]
out = {"source": "ncu --replay-mode application --cache-control none (kernels in step order, no flush between "
                  "them); bytes per step, mean over %d steps" % len(steps), "per_kernel": {}}
for key, frags in ROOF_KERNELS.items():
    tot = []
    for st in steps:
        tot.append(sum(x.get("dram__bytes_read.sum", 0) + x.get("dram__bytes_write.sum", 0)
                       for x in st if any(f in x["name"] for f in frags)))
    if tot and max(tot) > 0:
        out[key] = sum(tot) / len(tot)
for st in steps[-1:]:
    for x in st:
        out["per_kernel"][x["name"][:80]] = {"read": x.get("dram__bytes_read.sum"), "write": x.get("dram__bytes_write.sum"),
                                             "ns": x.get("gpu__time_duration.sum")}
path = os.path.join(REPO, "profiles", "ncu_traffic_instep.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "per_kernel"}, indent=1))
