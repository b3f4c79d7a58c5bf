"""Summarise ncu output into profiles/ (tracked).

  python tools/summarize_ncu.py --launches gpurun_out/launches.csv \
      --full gpurun_out/prof_full.ncu-rep --tag r01

Writes profiles/<tag>_launches.csv (raw launch list), profiles/<tag>_kernel_shares.md (per
kernel family: launches, total and mean device time, share of one mini-batch) and
profiles/<tag>_ncu_full.md (per captured launch: duration, DRAM bytes, tensor-pipe and
throughput percentages, registers, grid, dynamic smem).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import os
import re
import shutil
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def family(name: str) -> str:
    m = re.search(r"(gemm_bf16_2sm_kernel|gemm_bf16_tn_kernel)<(\d+), \(?(?:bool\))?(\d|true|false)\)?, "
                  r"\(?(?:bool\))?(\d|true|false)\)?(?:, \(?(?:bool\))?(\d|true|false)\)?)?", name)
    if m:
        kind, bn, a, b, sgd = m.groups()
        a = a in ("1", "true")
        b = b in ("1", "true")
        sgd = sgd in ("1", "true")
        role = "wgrad+sgd" if sgd else ("wgrad" if a and b else ("dgrad" if b else "fwd"))
        return f"{kind}<BN={bn}> [{role}]"
    for k in ("allreduce_sgd", "xent_kernel", "sum_rows", "gather_kernel", "gen_bf16", "gen_f64",
              "init_kernel", "ordered_sum", "linear_allreduce"):
        if k in name:
            return k
    return name[:60]


def launches(path: str, tag: str) -> None:
    shutil.copy(path, os.path.join(PROF, f"{tag}_launches.csv"))
    rows = []
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rdr = csv.DictReader(io.StringIO(text[start:]))
    for r in rdr:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r.get("Metric Unit", "")
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        rows.append((r["Kernel Name"], us))
    # one mini-batch = the launches between two consecutive gather kernels (last full one)
    idx = [i for i, (n, _) in enumerate(rows) if "gather_kernel" in n or "gather_inline_kernel" in n]
    step = rows[idx[-2]:idx[-1]] if len(idx) >= 2 else rows
    agg = collections.OrderedDict()
    for n, us in step:
        k = family(n)
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
    total = sum(t for _, t in agg.values())
    out = [f"# {tag}: kernel shares of one mini-batch (ncu launch list, cold-cache, serialised)\n",
           f"Source: `{os.path.basename(path)}` from `ncu --metrics gpu__time_duration.sum "
           f"--clock-control none` over `python tools/profile_step.py --size 65536` "
           f"(BASELINE configs[1] model, batch 512, N=1).  Absolute times are serialised "
           f"per-launch times; compare shares.\n",
           "| kernel family | launches / step | total us | mean us | share |",
           "|---|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {c} | {t:.1f} | {t / c:.1f} | {100 * t / total:.1f}% |")
    out.append(f"| **total** | {sum(c for c, _ in agg.values())} | {total:.1f} | | 100% |")
    with open(os.path.join(PROF, f"{tag}_kernel_shares.md"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


def full(path: str, tag: str, skip: str = "-s 75 -c 25") -> None:
    SKIP = skip
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, units = r[0], r[1]
    want = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
            ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
            ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
            ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"),
            ("launch__shared_mem_per_block_dynamic", "dyn smem")]
    idx = [(hdr.index(k), lab, units[hdr.index(k)]) for k, lab in want if k in hdr]
    ki = hdr.index("Kernel Name")
    out = [f"# {tag}: ncu --set full, one mini-batch (N=1, configs[1] model)\n",
           f"Source: `{os.path.basename(path)}` (`ncu --set full --clock-control none "
           f"--import-source on -k regex:\"gemm_bf16|allreduce_sgd|xent|gather\" {SKIP} "
           f"python tools/profile_step.py --size 65536`).  `traffic` per launch = DRAM read + "
           f"write.\n",
           "| # | kernel | " + " | ".join(f"{lab} ({u})" if u else lab for _, lab, u in idx) + " |",
           "|---|---|" + "---|" * len(idx)]
    for n, row in enumerate(r[2:]):
        out.append(f"| {n} | {family(row[ki])} | " + " | ".join(row[i] for i, _, _ in idx) + " |")
    with open(os.path.join(PROF, f"{tag}_ncu_full.md"), "w") as f:
        f.write("\n".join(out) + "\n")
    print("\n".join(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--skip", default="-s 75 -c 25", help="the ncu -s/-c flags of the capture")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    if a.full:
        full(a.full, a.tag, a.skip)


if __name__ == "__main__":
    main()
