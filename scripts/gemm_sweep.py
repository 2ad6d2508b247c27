"""Fixed-cost probe of the tcgen05 GEMM engine: back-to-back launches of one
shape, CUDA-event timed.  usage: python scripts/gemm_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo  # noqa: E402


def run(ctx, M, N, K, a_mn=False, b_mn=False, bn=128, splits=1, reps=50):
    a = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(torch.bfloat16)
    b = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda")
    lda = M if a_mn else K
    ldb = N if b_mn else K
    for _ in range(3):
        ctx.gemm(M, N, K, a, lda, a_mn, b, ldb, b_mn, out, N, bn=bn, splits=splits)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(100_000_000)  # the host enqueues every rep while the GPU sleeps
    e0.record()
    for _ in range(reps):
        ctx.gemm(M, N, K, a, lda, a_mn, b, ldb, b_mn, out, N, bn=bn, splits=splits)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    print(f"{M:6d}x{N:5d}x{K:6d} a_mn={int(a_mn)} b_mn={int(b_mn)} bn={bn:3d} s={splits:3d}: "
          f"{us:8.2f} us {2 * M * N * K / us / 1e6:8.1f} TF/s", flush=True)


def main():
    ctx = appo.Context(0)
    torch.cuda._sleep(10)
    if os.environ.get("SWEEP") == "infer":
        for bn in (64, 128, 256):
            run(ctx, 16384, 1536, 512, bn=bn, reps=20)
            run(ctx, 16384, 512, 2304, bn=bn, reps=20)
        return
    if os.environ.get("SWEEP") == "wgrad2":
        # round 2: split-K choices that fill 148 SMs in one wave (per-SM L2 intake bound)
        for bn, sp in ((64, 1), (128, 3), (64, 2), (256, 6), (128, 2)):
            run(ctx, 1536, 512, 2048, a_mn=True, b_mn=True, bn=bn, splits=sp)
        for bn, sp in ((64, 1), (128, 2), (256, 4), (192, 3)):
            run(ctx, 512, 2304, 2048, a_mn=True, b_mn=True, bn=bn, splits=sp)
        for bn, sp in ((64, 1), (128, 2), (256, 4)):
            run(ctx, 2112, 512, 2304, bn=bn, splits=sp)
        return
    if os.environ.get("SWEEP") == "wgrad":
        for bn, sp in ((256, 1), (256, 2), (256, 3), (128, 1), (128, 2), (128, 4), (64, 1)):
            run(ctx, 1536, 512, 2048, a_mn=True, b_mn=True, bn=bn, splits=sp)
        for bn, sp in ((256, 1), (128, 1), (128, 2), (64, 1), (64, 2), (192, 1)):
            run(ctx, 512, 2304, 2048, a_mn=True, b_mn=True, bn=bn, splits=sp)
        for bn, sp in ((256, 1), (128, 1), (64, 1)):
            run(ctx, 2112, 1536, 512, bn=bn, splits=sp)
        for bn, sp in ((128, 1), (64, 1), (256, 1)):
            run(ctx, 2048, 512, 1536, b_mn=True, bn=bn, splits=sp)
            run(ctx, 2048, 2304, 512, b_mn=True, bn=bn, splits=sp)
            run(ctx, 2112, 512, 2304, bn=bn, splits=sp)
        return
    run(ctx, 128, 128, 64)
    run(ctx, 128, 256, 512, bn=256)
    run(ctx, 2112, 1536, 512, bn=256)
    run(ctx, 2112, 512, 2304, bn=128)
    run(ctx, 2048, 512, 1536, b_mn=True, bn=128)
    run(ctx, 2048, 2304, 512, b_mn=True, bn=128)
    run(ctx, 1536, 512, 2048, a_mn=True, b_mn=True, bn=256, splits=3)
    run(ctx, 1536, 512, 2048, a_mn=True, b_mn=True, bn=256, splits=1)
    run(ctx, 512, 2304, 2048, a_mn=True, b_mn=True, bn=256, splits=1)
    run(ctx, 512, 2304, 2048, a_mn=True, b_mn=True, bn=128, splits=1)
    run(ctx, 8192, 8192, 8192, bn=256, reps=10)


if __name__ == "__main__":
    main()
