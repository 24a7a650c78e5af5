#!/usr/bin/env python3
"""Device time of one MRC step at configs[1]: CUDA-graph replay vs the same
sequence issued call by call (no per-phase events), L2 flushed before each.

  python tools/step_timing.py [--steps 20] [--config c1]
"""
import argparse
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--config", default="c1")
    args = ap.parse_args()
    import torch
    import paper_1810_03099_b200 as R
    from paper_1810_03099_b200 import corpus as C

    cp, cfg = C.config_corpus(args.config)
    thr = C.load_configs()["thresholds"]
    refs = C.sample_refs(cfg["ref_seed"], cp.n_docs, cfg["K"])
    tau = thr["tau_mrc"]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    ctx = R.Context(0)
    ctx.set_stream(stream.cuda_stream)
    ctx.load_corpus(cp.tokens, cp.doc_off, cp.vocab)
    flush = torch.empty(512 << 18, dtype=torch.int32, device=dev)

    def graph():
        ctx.mrc_step(refs, tau)

    def eager():
        ctx.count(R.WEIGHT_TFIDF)
        ctx.set_reference_docs(refs)
        ctx.sign(fetch=False)
        ctx.mrc_pairs_rows(tau, 0, cp.n_docs, fetch=False)

    out = {}
    with torch.cuda.stream(stream):
        for name, fn, collect in (("graph", graph, True), ("eager", eager, False)):
            for _ in range(3):
                flush.fill_(1)
                fn()
                if collect:
                    ctx.step_result()
            torch.cuda.synchronize()
            ts = []
            for s in range(args.steps):
                flush.fill_(s)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fn()
                b.record(stream)
                if collect:
                    ctx.step_result()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            out[name] = (float(np.median(ts)), float(np.min(ts)))
        ctx.set_profiling(True)
        for s in range(args.steps):
            flush.fill_(s)
            eager()
        torch.cuda.synchronize()
        ph = ctx.phase_times()
    print({k: f"median {v[0]*1e3:.1f} us, min {v[1]*1e3:.1f} us" for k, v in out.items()})
    print({k: f"{v[0] / args.steps * 1e3:.1f} us" for k, v in ph.items() if v[1]})


if __name__ == "__main__":
    main()
