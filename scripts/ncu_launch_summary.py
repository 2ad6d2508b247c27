"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into
per-kernel counts, total/avg device time and share (cold-cache, serialised
timings: compare SHARES with bench.py's live numbers, not absolutes).

usage: python scripts/ncu_launch_summary.py gpurun_out/launches.csv [--skip N]
"""
import collections
import csv
import re
import sys


AG_NAMES = {0: "gemm_bf16_tcgen05", 1: "gemm_conv_nhwc_gather_tcgen05",
            2: "gemm_conv1_u8_implicit_tcgen05", 3: "gemm_dgrad_implicit_tcgen05",
            4: "gemm_conv1_wgrad_implicit_tcgen05", 5: "gemm_conv_taps_implicit_tcgen05",
            6: "gemm_conv_taps_wgrad_tcgen05"}


# dedicated kernels: symbol -> the class name the library times them under
SYMBOL_CLASSES = {"conv1_s2d_kernel": "conv1_s2d_tcgen05",
                  "conv1_s2d_wgrad_kernel": "conv1_s2d_wgrad_tcgen05",
                  "conv2_s2d_kernel": "conv2_s2d_tcgen05",
                  "conv2_dgrad_kernel": "conv2_dgrad_s2d_tcgen05",
                  "gru_infer_fused_kernel": "gru_infer_fused_tcgen05",
                  "gru_g_fwd_kernel": "gru_seq_fwd_kernel",
                  "gru_g_bwd_kernel": "gru_seq_bwd_kernel"}


def kname(full: str) -> str:
    """Kernel class; GEMM engine instantiations by gather mode (the same names
    bench.py / the timing report use)."""
    m = re.search(r"gemm_bf16_kernel<([^>]*)>", full.replace("(int)", "").replace("(bool)", ""))
    if m:
        args = [a.strip() for a in m.group(1).split(",")]
        ag = int(args[4]) if len(args) > 4 and args[4].lstrip("-").isdigit() else 0
        return AG_NAMES.get(ag, "gemm_bf16_tcgen05")
    s = full
    if s.startswith("void "):
        s = s[5:]
    s = s.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    s = s.replace("appo_b200::", "")
    s = s.split("(")[0]
    s = re.sub(r"<.*", "", s)
    return SYMBOL_CLASSES.get(s, s)


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1 + skip:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3)
        a = agg[kname(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | avg us | share |")
    print(f"|---|---:|---:|---:|---:|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.1f} | {t / n:.2f} | {t / tot:.3f} |")
    print(f"\ntotal {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main()
