#!/usr/bin/env python3
"""CUPTI timeline (torch.profiler / Kineto) of one captured MRC step at a
config (default configs[1]): every kernel's start / end / stream relative to
the step's first kernel — the critical path of the graph replay."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1810_03099_b200 as R  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cp, cfg = C.config_corpus(name)
refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
tau = C.load_configs()["thresholds"]["tau_mrc"]
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
ctx = R.Context(0)
ctx.set_stream(stream.cuda_stream)
tok = torch.from_numpy(cp.tokens.view("int32")).to(dev)
flush = torch.empty(128 << 20, dtype=torch.int32, device=dev)
with torch.cuda.stream(stream):
    ctx.load_corpus_device(tok.data_ptr(), cp.doc_off, cp.vocab)
    for _ in range(4):
        ctx.mrc_step(refs, tau, R.WEIGHT_TFIDF, 0, cp.n_docs)
        ctx.step_result()
    torch.cuda.synchronize(dev)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            flush.fill_(1)
            ctx.mrc_step(refs, tau, R.WEIGHT_TFIDF, 0, cp.n_docs)
            ctx.step_result()
    torch.cuda.synchronize(dev)
path = os.path.join(REPO, "gpurun_out", f"step_trace_{name}.json")
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
# the last step: kernels after the last fill (elementwise) kernel
last_fill = max(i for i, e in enumerate(ev) if "fill" in e["name"].lower() or "elementwise" in e["name"].lower())
step = ev[last_fill + 1:]
t0 = step[0]["ts"]
for e in step:
    nm = e["name"].replace("refsig_gpu::(anonymous namespace)::", "").replace("refsig_gpu::", "")[:44]
    print(f"{e['ts'] - t0:8.1f} {e['ts'] + e['dur'] - t0:8.1f} {e['dur']:7.1f}  s={e.get('args', {}).get('stream')}  {nm}")
print(f"step span {step[-1]['ts'] + step[-1]['dur'] - t0:.1f} us")
