"""Times the tcgen05 GEMM engine on the model's shapes (CUDA events, warm L2
excluded by >L2 operands where possible) and reports TFLOP/s and effective
GB/s.  usage: python scripts/gemm_bench.py [shape-name ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_11751_b200 as appo  # noqa: E402

# name: (M, N, K, a_mn, b_mn, out_bf16, bn, splits)
SHAPES = {
    "conv2_dcol": (200704, 512, 64, False, True, True, 256, 1),
    "conv3_dcol": (36864, 576, 128, False, True, True, 192, 1),
    "gi_infer": (16384, 1536, 512, False, False, False, 256, 1),
    "conv1_fwd": (1113024, 32, 192, False, False, True, 32, 1),
    "conv2_fwd": (206976, 64, 512, False, False, True, 64, 1),
    "conv3_fwd": (294912, 128, 576, False, False, True, 128, 1),
    "fc_fwd": (16384, 512, 2304, False, False, True, 128, 1),
    "big_square": (8192, 8192, 8192, False, False, False, 256, 1),
}


def run(name, ctx, iters=10):
    M, N, K, amn, bmn, obf, bn, sp = SHAPES[name]
    A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if obf else torch.float32)
    lda = M if amn else K
    ldb = N if bmn else K
    flags = appo.EPI_BF16 if obf else 0
    for _ in range(2):
        ctx.gemm(M, N, K, A, lda, amn, B, ldb, bmn, out, N, flags=flags, bn=bn, splits=sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        ctx.gemm(M, N, K, A, lda, amn, B, ldb, bmn, out, N, flags=flags, bn=bn, splits=sp)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = 2.0 * M * N * K
    byts = 2 * (M * K + N * K) + M * N * (2 if obf else 4)
    print(f"{name:12s} {M}x{N}x{K} bn{bn} s{sp}: {ms * 1e3:8.1f} us  "
          f"{flops / ms / 1e9:7.1f} TF/s  {byts / ms / 1e6:7.1f} GB/s", flush=True)


def main():
    ctx = appo.Context(0)
    names = sys.argv[1:] or list(SHAPES)
    for n in names:
        run(n, ctx)


if __name__ == "__main__":
    main()
