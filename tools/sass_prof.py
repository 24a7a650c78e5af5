#!/usr/bin/env python3
"""Per-SASS-instruction executed counts and stall samples from an ncu report
(the --page source view), sorted by executed warp instructions.

  python tools/sass_prof.py gpurun_out/prof.ncu-rep [--top 40] [--kernel regex]"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--order", choices=["addr", "count"], default="count")
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = rows[0]
    ia, isrc, iex, ism = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
        h.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[1:]:
        try:
            recs.append((r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ism] or 0)))
        except (ValueError, IndexError):
            pass
    tot = sum(x[2] for x in recs) or 1
    tots = sum(x[3] for x in recs) or 1
    print(f"total executed warp instructions {tot:.4g}, stall samples {tots}")
    sel = sorted(recs, key=lambda x: -x[2])[: args.top] if args.order == "count" else recs
    for a, src, n, smp in sel:
        print(f"{a[-5:]} {n:>12d} {100 * n / tot:5.1f}% {100 * smp / tots:5.1f}%s  {src}")


if __name__ == "__main__":
    main()
