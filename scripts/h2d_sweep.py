"""Host->device copy throughput on this box: chunk size, number of concurrent
copy streams, and with a concurrent HBM-heavy kernel (the e2e arm's situation).
usage: python scripts/h2d_sweep.py"""
import torch

GB = 1e9
n, od = 8192, 27648  # one env group's observations (226 MB)
host = [torch.empty(n * od, dtype=torch.uint8).pin_memory() for _ in range(4)]
dev = [torch.empty(n * od, dtype=torch.uint8, device="cuda") for _ in range(4)]
big = torch.empty(2 * 1024 ** 3, dtype=torch.uint8, device="cuda")


def run(nstreams, reps=8, chunk=None, load=False):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    ls = torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    if load:
        with torch.cuda.stream(ls):
            for _ in range(40):
                big.add_(1)
    total = 0
    for r in range(reps):
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                k = (r * nstreams + i) % 4
                if chunk:
                    for o in range(0, n * od, chunk):
                        dev[k][o:o + chunk].copy_(host[k][o:o + chunk], non_blocking=True)
                else:
                    dev[k].copy_(host[k], non_blocking=True)
                total += n * od
    for s in streams:
        ev = torch.cuda.Event()
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return total / (e0.elapsed_time(e1) * 1e-3) / GB


run(1, 2)
for ns in (1, 2, 4):
    print(f"streams={ns} whole 226MB copies: {run(ns):6.1f} GB/s   with HBM load: {run(ns, load=True):6.1f} GB/s")
for ch in (4 << 20, 32 << 20):
    print(f"streams=2 chunks of {ch >> 20} MB: {run(2, chunk=ch):6.1f} GB/s")
