"""Per-kernel-class summary of an ncu metrics CSV (scripts/gpu_evidence.sh:
sm__pipe_tensor_cycles_active, sm__throughput, DRAM bytes, duration over one
inference step of 16,384 envs + 8 learner steps).  Kernels are grouped by
name + launch shape label so the inference and learner launches of the same
template stay apart (GEMM shapes differ by grid).  Writes markdown.

    python scripts/tensor_pipe_summary.py gpurun_out/tensor_pipe.csv > profiles/r02_tensor_pipe.md
"""
import collections
import csv
import re
import sys


def short(name):
    m = re.search(r"::(\w+)(<[^(]*>)?\(", name)
    if not m:
        return name[:40]
    # GEMM engine variants differ by template (tile width, operand majors,
    # A-operand generator: plain / conv1 u8 / conv taps / wgrad / dgrad)
    return m.group(1) + (m.group(2) or "").replace(" ", "")


def main(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Grid Size",
                                    "Block Size")}
    launches = collections.OrderedDict()
    for r in rows[i + 1:]:
        if len(r) != len(hdr):
            continue
        key = int(r[ix["ID"]])
        d = launches.setdefault(key, {"name": short(r[ix["Kernel Name"]]),
                                      "grid": r[ix["Grid Size"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    groups = collections.OrderedDict()
    for d in launches.values():
        g = groups.setdefault((d["name"], d["grid"]), [])
        g.append(d)
    tot = sum(d["gpu__time_duration.sum"] for d in launches.values())
    print("| kernel | grid | launches | avg us | share | tensor pipe % (elapsed) | "
          "tensor pipe % (active SMs) | SM throughput % | DRAM MB/launch | DRAM GB/s |")
    print("|---|---|---:|---:|---:|---:|---:|---:|---:|---:|")
    for (name, grid), ds in sorted(groups.items(), key=lambda kv: -sum(
            d["gpu__time_duration.sum"] for d in kv[1])):
        n = len(ds)
        t = sum(d["gpu__time_duration.sum"] for d in ds) / n
        mb = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds) / n / 1e6
        te = sum(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"] for d in ds) / n
        ta = sum(d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"] for d in ds) / n
        sm = sum(d["sm__throughput.avg.pct_of_peak_sustained_elapsed"] for d in ds) / n
        print(f"| {name} | {grid} | {n} | {t / 1e3:.1f} | {t * n / tot:.3f} | {te:.1f} | {ta:.1f} | "
              f"{sm:.1f} | {mb:.1f} | {mb * 1e6 / t:.0f} |")
    print(f"\ntotal {tot / 1e3:.1f} us over {len(launches)} launches (ncu serialised, cold caches)")


if __name__ == "__main__":
    main(sys.argv[1])
