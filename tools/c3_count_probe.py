#!/usr/bin/env python3
"""configs[3] K1 count: phase time of repeated counts (first = cold) and the
document-length classes (how many documents / tokens take each K1 path)."""
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_03099_b200 as R  # noqa: E402
from paper_1810_03099_b200 import corpus as C  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cp, cfg = C.config_corpus(cfg_name)
lens = np.diff(cp.doc_off).astype(np.int64)
edges = [0, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 1 << 40]
cls = {f"{edges[i] + 1}..{edges[i + 1]}": [int(((lens > edges[i]) & (lens <= edges[i + 1])).sum()),
                                           int(lens[(lens > edges[i]) & (lens <= edges[i + 1])].sum())]
       for i in range(len(edges) - 1)}
dev = torch.device("cuda", 0)
flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)
out = {"config": cfg_name, "docs": int(cp.n_docs), "tokens": int(cp.doc_off[-1]), "max_len": int(lens.max()),
       "classes_docs_tokens": cls, "count_ms": []}
with R.Context(0) as ctx:
    stream = torch.cuda.Stream(dev)
    ctx.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
        for r in range(reps):
            flush.fill_(r)
            ctx.set_profiling(True)
            ctx.count(R.WEIGHT_TFIDF)
            torch.cuda.synchronize(dev)
            out["count_ms"].append(ctx.phase_times()["count"][0])
            ctx.set_profiling(False)
print(json.dumps(out))
