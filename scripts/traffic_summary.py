"""ncu CSV (dram bytes + duration per launch) -> per-kernel-class summary.
usage: python scripts/traffic_summary.py launches.csv > profiles/traffic.json"""
import csv
import json
import re
import sys
from collections import defaultdict

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


def klass(name):
    m = re.search(r"gemm_bf16_kernel<[^>]*?(\d+)\s*>", name.replace("(int)", "").replace("(bool)", ""))
    if "gemm_bf16_kernel" in name and m:
        return AG_NAMES.get(int(m.group(1)), "gemm_bf16_tcgen05")
    base = re.sub(r"^void\s+", "", name)
    base = base.split("(")[0] if not base.startswith("(") else base
    base = base.replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    base = re.sub(r"<.*", "", base).split("::")[-1]
    return SYMBOL_CLASSES.get(base, base)


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "us": 0.0})
    launches = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        name, metric, unit = d["Kernel Name"], d["Metric Name"], d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        key = (d["ID"], name)
        if metric.startswith("dram__bytes"):
            scale = {"byte": 1, "B": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6,
                     "Gbyte": 1e9, "GB": 1e9}.get(unit, 1)
            per[klass(name)]["dram_bytes"] += v * scale
        elif metric == "gpu__time_duration.sum":
            scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
                     "ms": 1e3, "msecond": 1e3}.get(unit, 1)
            per[klass(name)]["us"] += v * scale
            per[klass(name)]["launches"] += 1
            launches.append((d["ID"], klass(name), v * scale))
    out = {}
    for k, s in per.items():
        n = max(s["launches"], 1)
        out[k] = s["dram_bytes"] / n
    json.dump({"traffic_bytes_per_launch": out,
               "detail": {k: {"launches": s["launches"], "dram_bytes_total": s["dram_bytes"],
                              "us_total": s["us"]} for k, s in per.items()},
               "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                         "gpu__time_duration.sum --clock-control none over "
                         "scripts/traffic_step.py (1 inference step of 16384 envs + 8 learner "
                         "steps of 2048 samples = the bench's 32:256 launch mix); "
                         "cold-cache serialized replays"},
              sys.stdout, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1])
