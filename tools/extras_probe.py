#!/usr/bin/env python3
"""Run bench.py's configs[4] extra alone (and optionally after configs[3]) to
isolate cross-measurement effects.  python tools/extras_probe.py [c4|c3c4|c4prof]"""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402

import bench  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "c4"
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
if mode == "c3c4":
    r = bench.measure_c3(dev)
    print("c3", json.dumps({k: r[k] for k in ("candidates",)}), flush=True)
r = bench.measure_c4(dev)
print(mode, json.dumps({k: r.get(k) for k in ("ms_per_batch", "ms_each_batch", "wall_ms_per_batch", "host_ms_per_call",
                                               "phase_ms_per_batch")}), flush=True)
