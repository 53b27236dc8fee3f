"""Per-launch time of the tcgen05 GEMM engine for small learner-step shapes
(CUDA graph of back-to-back launches, CUDA events) — the engine's latency floor."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1910_06591_b200 as S

shapes = [(128, 128, 64, 128, 1), (672, 1024, 64, 128, 1), (672, 1024, 288, 128, 1),
          (672, 256, 2592, 128, 10), (672, 256, 2592, 128, 1), (1024, 544, 672, 128, 4),
          (1024, 544, 672, 128, 1), (4096, 4096, 4096, 256, 1)]
for (M, N, K, bn, sp) in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda")
    S.debug_gemm(A, B, bn=bn, splits=sp, out=D)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    err = ((D - ref).norm() / ref.norm()).item()
    s = torch.cuda.Stream()
    reps = 20
    with torch.cuda.stream(s):
        S.debug_gemm(A, B, bn=bn, splits=sp, out=D, stream=s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                S.debug_gemm(A, B, bn=bn, splits=sp, out=D, stream=s)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / reps
    print(f"M={M} N={N} K={K} bn={bn} splits={sp}: {us:8.2f} us/launch  "
          f"{2*M*N*K/us/1e6:8.1f} TF/s  relerr {err:.1e}")
