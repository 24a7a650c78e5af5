#!/usr/bin/env python3
"""Summarise `ncu --page source --csv` (SASS view) output: instruction counts
and stall samples per opcode and the hottest instructions, per kernel.
  ncu -i rep --page source --csv --kernel-name regex:K ... > x.csv; python tools/sass_hot.py x.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
blocks = []
for i, r in enumerate(rows):
    if r and r[0] == "Kernel Name":
        blocks.append((r[1], i))
blocks.append((None, len(rows)))
for (name, s), (_, e) in zip(blocks, blocks[1:]):
    hdr = rows[s + 1]
    idx = {h: k for k, h in enumerate(hdr)}
    byop, stall, top, tot = collections.Counter(), collections.Counter(), [], 0
    for r in rows[s + 2:e]:
        if len(r) < len(hdr):
            continue
        ie = float(r[idx["Instructions Executed"]] or 0)
        st = float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        src = r[idx["Source"]].split()
        op = (src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "?"))
        byop[op] += ie
        stall[op] += st
        tot += ie
        top.append((st, ie, r[idx["Address"]][-5:], r[idx["Source"]][:80]))
    print("=" * 8, name[:100], "instructions", int(tot))
    print("by opcode (inst):", [(o, int(c)) for o, c in byop.most_common(12)])
    print("by opcode (stall samples):", [(o, int(c)) for o, c in stall.most_common(10)])
    top.sort(reverse=True)
    for t in top[:top_n]:
        print("  stall %6d  inst %9d  %s  %s" % t)
