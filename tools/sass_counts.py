"""SASS evidence for the hot kernels of libedl_b200.so (cuobjdump -sass): per kernel the
count of tcgen05 / TMA / TMEM instructions that prove the sm_100a path (UTCHMMA = tcgen05.mma,
UTCBAR = tcgen05.commit, UTMALDG / UTMASTG / UTMAPF = TMA tensor load / store / prefetch,
UBLKCP / UBLKPF = bulk copy / prefetch, LDTM = tcgen05.ld, SYNCS = mbarrier ops) and the
local-memory traffic that would reveal register spills (LDL / STL).

    python tools/sass_counts.py [--lib paper_1909_11985_b200/libedl_b200.so] > profiles/r02_sass_counts.md
"""
import argparse
import collections
import os
import re
import subprocess

OPS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UTMAPF", "UBLKCP", "UBLKPF", "LDTM",
       "SYNCS", "LDL", "STL"]
HOT = [
    ("gemm_bf16_2sm_kernel<128, false, false, false, 2, 1, false, 0, false>", "fwd GEMM (K-major A/B, A multicast)"),
    ("gemm_bf16_2sm_kernel<128, false, true, false, 2, 1, false, 0, false>", "dgrad GEMM (MN-major B, A multicast)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, false, 1, false>", "wgrad + fused SGD, split master (N=1 dominant)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, false, 2, false>", "wgrad + fused SGD, split in / fp32 out (before a switch)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, false, 3, false>", "wgrad + fused SGD, fp32 in / split out (after a switch)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, false, 1, true>", "wgrad + fused SGD, split master, A resident (opt-in)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, false, 0, false>", "wgrad + fused SGD, fp32 master"),
    ("gemm_bf16_2sm_kernel<128, true, true, false, 1, 1, false, 0, false>", "wgrad (N>1, reduce-scatter routed)"),
    ("gemm_bf16_2sm_kernel<128, true, true, true, 1, 1, true, 0, false>", "wgrad + fused exchange (mode 4)"),
    ("push_allreduce_sgd_kernel<false>", "push all-gather + sharded SGD (N>1)"),
    ("push_allreduce_sgd_kernel<true>", "push all-gather + sharded SGD + momentum"),
    ("xent_kernel<16>", "softmax-CE + loss sum"),
    ("gather_inline_kernel", "leased-run gather"),
    ("master_split_kernel", "split master: fp32 -> (W, lo)"),
    ("master_join_kernel", "split master: (W, lo) -> fp32"),
    ("wgrad_sgd_bres_kernel", "B-resident wgrad + SGD (opt-in)"),
    ("bwd_pair_kernel", "dgrad l-1 + wgrad/SGD l pair (opt-in)"),
]


def main():
    ap = argparse.ArgumentParser()
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ap.add_argument("--lib", default=os.path.join(root, "paper_1909_11985_b200", "libedl_b200.so"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True).stdout
    dem = subprocess.run(["c++filt"], input=sass, capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for ln in dem.splitlines():
        m = re.match(r"\s+Function : (.*)", ln)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", ln)
        if m:
            op = m.group(1).split(".")[0]
            funcs[cur][op] += 1
    print("# SASS instruction counts of the hot kernels (cuobjdump -sass, sm_100a)\n")
    print(f"`python tools/sass_counts.py` on `{os.path.relpath(a.lib, root)}`.  Static counts"
          " (instructions in the binary, not executions).\n")
    print("| kernel | role | " + " | ".join(OPS) + " |")
    print("|---|---|" + "---|" * len(OPS))
    for pat, role in HOT:
        hits = [f for f in funcs if pat in f]
        if not hits:
            continue
        c = funcs[hits[0]]
        print(f"| `{pat}` | {role} | " + " | ".join(str(c.get(o, 0)) for o in OPS) + " |")


if __name__ == "__main__":
    main()
