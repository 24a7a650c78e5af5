#!/usr/bin/env python3
"""Summarise ncu output into profiles/ (run here, after gpurun brings the
reports back).

  python tools/ncu_summary.py --launches gpurun_out/launches_bench.csv \
      --full gpurun_out/prof_r01_full.ncu-rep --tag r01

Writes profiles/ncu_launches_<tag>.csv (the raw launch list),
profiles/ncu_launches_<tag>.md (per-kernel share of one timed step),
profiles/ncu_full_<tag>.md (per-kernel metrics of the --set full capture) and
profiles/ncu_traffic.json (per-launch DRAM bytes read+write, used by bench.py's
roofline.traffic).
"""
import argparse
import collections
import csv
import json
import os
import shutil
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

# bench.py roofline keys -> kernel name fragments
ROOF_KERNELS = {"mrc_tiles": ["mrc_tc_kernel", "tc_forms_kernel"], "sign": ["sign_kernel"], "pair_emit": ["emit_kernel"],
                "count": ["count_warp_kernel", "group_sort_kernel", "group_split_kernel", "count_large_kernel", "idf_kernel"],
                "reference": ["ref_build_kernel"],
                "simhash": ["simhash_kernel"], "hamming_tiles": ["hamming_bitmap_kernel"]}


def short(name):
    n = name.replace("refsig_gpu::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    return n.split("(")[0]


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hdr = None
    recs = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"])
                if d.get("Metric Unit") == "ns":
                    v /= 1000.0
                elif d.get("Metric Unit") == "ms":
                    v *= 1000.0
                recs.append((int(d["ID"]), short(d["Kernel Name"]), v))
    shutil.copy(path, os.path.join(PROF, f"ncu_launches_{tag}.csv"))
    # the last complete step: take the tail after the last merge->mrc sequence; simpler: per-kernel mean
    by = collections.defaultdict(list)
    for _, k, v in recs:
        by[k].append(v)
    total = sum(sum(v) for v in by.values())
    lines = [f"# ncu launch list ({tag}) — `--metrics gpu__time_duration.sum --clock-control none`",
             "", "Serialised, cold-cache per-launch device times (compare shares, not absolutes).",
             f"{len(recs)} launches, {total:.1f} us total.", "",
             "| kernel | launches | mean us | total us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {sum(v):.1f} | {sum(v) / total:.1%} |")
    # one MRC step: every distinct step kernel once (mean of its launches)
    step = {k: sum(v) / len(v) for k, v in by.items() if any(f in k for f in STEP_KERNELS)}
    st = sum(step.values())
    lines += ["", f"## One MRC step (configs[1]): {len(step)} kernels, {st:.1f} us serialised", "",
              "Each step kernel's mean launch time and its share of the serialised step (the K1 classes run "
              "concurrently on side streams in the real step, so their share is an upper bound).", "",
              "| kernel | mean us | share of step |", "|---|---:|---:|"]
    for k, v in sorted(step.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {v:.1f} | {v / st:.1%} |")
    open(os.path.join(PROF, f"ncu_launches_{tag}.md"), "w").write("\n".join(lines) + "\n")


STEP_KERNELS = ["count_warp_kernel", "group_sort_kernel", "group_split_kernel", "count_large_kernel", "idf_kernel", "ref_build_kernel", "sign_kernel", "sign_col_kernel", "tc_forms_kernel",
                "mrc_tc_kernel", "mrc_bitmap_kernel2", "scan_small_kernel", "emit_kernel"]

WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
        ("smsp__inst_executed.sum", "warp inst"), ("lts__t_sector_hit_rate.pct", "L2 hit %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("sm__ops_path_tensor_src_fp16_dst_fp32.sum", "tensor fp16->fp32 ops")]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def full(path, tag, title=None, append=False, write_traffic=True):
    if path.endswith(".csv"):  # `ncu -i rep --page raw --csv` output made on the GPU box
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if "issue_stalled" in h and h.endswith("per_issue_active.ratio")]
    lines = ([f"## {title}", ""] if append else
             [f"# ncu --set full ({tag}) — per-kernel metrics", "",
              "Captured with `--set full --clock-control none --import-source on`; one launch per kernel of "
              "tools/prof_all.py (see each section). DRAM bytes are cold-cache (ncu flushes caches between "
              "replays).", ""] + ([f"## {title}", ""] if title else []))
    per_kernel = collections.defaultdict(list)  # kernel name -> [bytes per launch]
    per_inst = collections.defaultdict(list)  # kernel name -> [warp instructions per launch]
    for r in rows[2:]:
        k = short(r[idx["Kernel Name"]])
        lines.append(f"### `{k}`")
        for m, label in WANT:
            if m in idx:
                lines.append(f"- {label}: {r[idx[m]]} {units[idx[m]]}")
        top = sorted(stall, key=lambda h: -float(r[idx[h]] or 0))[:4]
        lines.append("- top stalls (warps per issue): " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}="
            f"{float(r[idx[h]] or 0):.1f}" for h in top))
        lines.append("")
        rd = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        per_kernel[k].append(rd + wr)
        if "smsp__inst_executed.sum" in idx:
            per_inst[k].append(float(r[idx["smsp__inst_executed.sum"]].replace(",", "")))
    # per step: each distinct kernel of a group once (mean over its captured launches)
    traffic = {}
    for k, v in per_kernel.items():
        for key, frags in ROOF_KERNELS.items():
            if any(f in k for f in frags) and not (key == "simhash" and "text_" in k):
                traffic[key] = traffic.get(key, 0.0) + sum(v) / len(v)
    open(os.path.join(PROF, f"ncu_full_{tag}.md"), "a" if append else "w").write("\n".join(lines) + "\n")
    if write_traffic:
        json.dump({k: v for k, v in traffic.items()}, open(os.path.join(PROF, "ncu_traffic.json"), "w"), indent=1)
        inst = {}
        for k, v in per_inst.items():
            for key, frags in ROOF_KERNELS.items():
                if any(f in k for f in frags) and not (key == "simhash" and "text_" in k):
                    inst[key] = inst.get(key, 0.0) + sum(v) / len(v)
        json.dump(inst, open(os.path.join(PROF, "ncu_inst.json"), "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--title", default=None)
    ap.add_argument("--append", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    if a.full:
        full(a.full, a.tag, a.title, a.append, not a.no_traffic)


if __name__ == "__main__":
    main()
