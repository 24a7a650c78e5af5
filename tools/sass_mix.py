#!/usr/bin/env python3
"""Opcode mix (executed warp instructions) per kernel of an ncu report's
source page.  python tools/sass_mix.py rep.ncu-rep [--top 20]"""
import argparse, csv, io, subprocess
from collections import Counter, OrderedDict

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=20)
args = ap.parse_args()
out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
blocks, cur = OrderedDict(), None
for ln in out:
    if ln.startswith('"Kernel Name"'):
        cur = ln.split('","')[1].split("(")[0].replace("void refsig_gpu::<unnamed>::", "")
        blocks.setdefault(cur, [])
        continue
    if cur:
        blocks[cur].append(ln)
for name, lines in blocks.items():
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    isrc, iex = h.index("Source"), h.index("Instructions Executed")
    c, tot = Counter(), 0
    for r in rows[1:]:
        try:
            n = int(r[iex] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[isrc].strip().split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        c[op.split(".")[0]] += n
        tot += n
    print(f"== {name}: {tot:.4g} warp instructions (both launches)")
    print("   " + "  ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(args.top)))
