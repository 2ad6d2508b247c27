"""Summarise an `ncu --set full` capture of one learner step
(scripts/gpu_ncu_learner.sh) into a per-kernel markdown table."""
import csv, io, subprocess, sys

rep = sys.argv[1]
# launch order of one Doom-shape learner step (model.cu learner_submit_impl)
ROLES = ["slot gather", "conv1 fwd", "conv2 fwd", "conv3 fwd", "FC fwd", "GRU input projection",
         "GRU fwd", "loss block", "head-gradient reduce", "GRU BPTT", "dW_ih", "dW_hh",
         "dx = dgi W_ih", "FC wgrad", "FC dgrad", "conv3 wgrad", "split-K reduce (conv3 wgrad)",
         "conv3 dgrad", "conv2 wgrad", "split-K reduce (conv2 wgrad)", "conv2 dgrad",
         "conv1 wgrad", "split-K reduce (conv1 wgrad)", "global norm", "Adam",
         "publish derived operands"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, rows = rows[0], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cols = [("us", "gpu__time_duration.sum", 1.0),
        ("DRAM MB rd", "dram__bytes_read.sum", 1.0),
        ("DRAM MB wr", "dram__bytes_write.sum", 1.0),
        ("grid", "launch__grid_size", 1.0),
        ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1.0),
        ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0)]
print(f"ncu --set full --clock-control none (cold caches, serialised launches): {rep}\n")
print("| # | kernel | " + " | ".join(c[0] for c in cols) + " |")
print("|---|---|" + "---:|" * len(cols))
tot = 0.0
for k, r in enumerate(rows):
    name = r[ix["Kernel Name"]].split("(")[0]
    for junk in ("appo_b200::", "<unnamed>::", "unnamed>::", "void "):
        name = name.replace(junk, "")
    if len(rows) == len(ROLES):
        name += f" ({ROLES[k]})"
    vals = []
    for _, key, _ in cols:
        v = r[ix[key]] if key in ix else ""
        try:
            f = float(v.replace(",", ""))
            vals.append(f"{f:.1f}" if key != "launch__grid_size" else str(int(f)))
        except ValueError:
            vals.append(v)
    tot += float(r[ix["gpu__time_duration.sum"]].replace(",", ""))
    print(f"| {k} | `{name}` | " + " | ".join(vals) + " |")
print(f"\nsum of kernel durations: {tot:.1f} us")
