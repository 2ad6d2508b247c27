"""Summarise an ncu --set full report: key throughput metrics, barrier waits and
the hottest SASS instructions with their top stall reasons.
usage: python scripts/ncu_hot.py report.ncu-rep [n_top]"""
import csv
import subprocess
import sys


def I(s):
    try:
        return int(s)
    except ValueError:
        return 0


def main():
    rep = sys.argv[1]
    ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                         capture_output=True, text=True).stdout.splitlines()))
    h, v = raw[0], raw[2]
    keys = ("gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__warps_eligible.avg.per_cycle_active", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    for i, n in enumerate(h):
        if n in keys:
            print(f"{n:70s} {v[i]}")
    src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                                          "--print-source=cuda,sass"],
                                         capture_output=True, text=True).stdout.splitlines()))
    hdr = [r for r in src if r and r[0] == "Line No"][0]
    names = hdr[32:49]
    seen, sass = set(), []
    for r in src:
        if len(r) > 40 and r[0] == "" and r[2].startswith("0x") and r[2] not in seen:
            seen.add(r[2])
            sass.append(r)
    sass.sort(key=lambda r: int(r[2], 16))
    tot = sum(I(r[4]) for r in sass) or 1
    print(f"stall samples {tot}")
    hot = sorted(sass, key=lambda r: -I(r[4]))[:ntop]
    hot_set = {r[2] for r in hot}
    for r in sass:
        if r[2] in hot_set or "TRYWAIT" in r[3]:
            st = sorted([(I(r[32 + i]), names[i]) for i in range(len(names))], reverse=True)[:2]
            print(f"{r[2][-5:]} {r[3][:64]:64s} exec={I(r[7]):9d} samp={100 * I(r[4]) / tot:5.1f}% "
                  f"{st[0][1]}:{st[0][0]} {st[1][1]}:{st[1][0]}")


if __name__ == "__main__":
    main()
