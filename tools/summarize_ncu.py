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
    name = re.sub(r"\((?:int|bool)\)", "", name)  # ncu's "(int)128, (bool)1" spelling
    m = re.search(r"(gemm_bf16_2sm_kernel|gemm_bf16_tn_kernel)<(\d+), (\d|true|false), "
                  r"(\d|true|false)(?:, (\d|true|false))?", name)
    if m:
        kind, bn, a, b, sgd = m.groups()
        a = a in ("1", "true")
        b = b in ("1", "true")
        sgd = sgd in ("1", "true")
        role = "wgrad+sgd" if sgd else ("wgrad" if a and b else ("dgrad" if b else "fwd"))
        targs = re.search(r"gemm_bf16_2sm_kernel<([^>]*)>", name)
        args = [a.strip() for a in targs.group(1).split(",")] if targs else []
        lo = args[7] if len(args) > 7 else "0"
        if sgd and lo != "0":
            role += {"1": ", split master", "2": ", split in / fp32 out",
                     "3": ", fp32 in / split out"}.get(lo, "")
            if len(args) > 8 and args[8] in ("1", "true"):
                role += ", A resident"
        return f"{kind}<BN={bn}> [{role}]"
    for k in ("allreduce_sgd", "xent_kernel", "sum_rows", "gather_kernel", "gen_bf16", "gen_f64",
              "init_kernel", "ordered_sum", "linear_allreduce"):
        if k in name:
            return k
    return name[:60]


def launches(path: str, tag: str) -> None:
    shutil.copy(path, os.path.join(PROF, f"{tag}_launches.csv"))
    rows = []
    dram = collections.defaultdict(lambda: [0.0, 0.0])  # launch ID -> [read MB, write MB]
    with open(path) as f:
        text = f.read()
    start = text.find('"ID"')
    rdr = csv.DictReader(io.StringIO(text[start:]))
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "KB": 1e-3, "MB": 1.0,
             "GB": 1e3, "B": 1e-6}
    for r in rdr:
        name = r.get("Metric Name")
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except (ValueError, KeyError):
            continue
        unit = r.get("Metric Unit", "")
        if name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram[r["ID"]][0 if name.endswith("read.sum") else 1] += v * scale.get(unit, 1e-6)
            continue
        if name != "gpu__time_duration.sum":
            continue
        us = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)
        rows.append((r["Kernel Name"], us, r["ID"]))
    # one mini-batch = the launches between two consecutive gather kernels (last full one)
    idx = [i for i, (n, _, _) in enumerate(rows) if "gather_kernel" in n or "gather_inline_kernel" in n]
    step = rows[idx[-2]:idx[-1]] if len(idx) >= 2 else rows
    agg = collections.OrderedDict()
    agg_dram = collections.OrderedDict()
    for n, us, lid in step:
        k = family(n)
        c, t = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, t + us)
        rd, wr = agg_dram.get(k, (0.0, 0.0))
        agg_dram[k] = (rd + dram[lid][0], wr + dram[lid][1])
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
    if dram:
        out += ["", "## DRAM traffic over one mini-batch (`--cache-control none`: caches not "
                "flushed between kernels, so dirty lines a kernel leaves in L2 are counted where "
                "they are written back; the sum over the mini-batch is the true HBM traffic)", "",
                "| kernel family | launches | us (serialised) | DRAM read MB | DRAM write MB |",
                "|---|---|---|---|---|"]
        for k, (c, t) in agg.items():
            rd, wr = agg_dram[k]
            out.append(f"| {k} | {c} | {t:.1f} | {rd:.1f} | {wr:.1f} |")
        trd = sum(v[0] for v in agg_dram.values())
        twr = sum(v[1] for v in agg_dram.values())
        out.append(f"| **total** | | | **{trd:.1f}** | **{twr:.1f}** |")
        out.append(f"\nMeasured HBM traffic per mini-batch: {(trd + twr) / 1e3:.2f} GB read + write.")
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
