"""Standalone tcgen05 engine timing (seed_debug_gemm)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1910_06591_b200 as S

def bench(M, N, K, bn, splits=1, it=20):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda")
    for _ in range(3):
        S.debug_gemm(A, B, bn=bn, splits=splits, out=D)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(it):
        S.debug_gemm(A, B, bn=bn, splits=splits, out=D)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / it
    tf = 2 * M * N * K / us / 1e6
    print(f"M={M} N={N} K={K} bn={bn} splits={splits}: {us:9.2f} us  {tf:8.2f} TFLOP/s", flush=True)

bench(4096, 4096, 4096, 256)
bench(4096, 4096, 4096, 128)
bench(8192, 8192, 8192, 256, it=5)
bench(268800, 16, 256, 16)
bench(268800, 16, 512, 16)
bench(268800, 16, 64, 16)
bench(148 * 128, 16, 64, 16)
bench(148 * 128, 16, 640, 16)
bench(148 * 128, 16, 64 * 40, 16)
bench(148 * 128, 256, 64 * 40, 256)
bench(4096, 4096, 4096, 256, splits=-1)
bench(268800, 16, 512, 16, splits=-1)
