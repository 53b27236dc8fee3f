"""Cycle stamps of CTA 0 of the tcgen05 GEMM engine (diagnostic build, see
probe_lstm.py --build): setup, producer issue, first full stage, MMA commit,
epilogue start / end, exit."""
import ctypes as C
import os
import sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "paper_1910_06591_b200", "libseed_prof.so")
os.environ["SEED_LIB"] = PROF
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402
lib = C.CDLL(PROF)
for (M, N, K) in [(128, 128, 64), (672, 1024, 288)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda")
    for _ in range(3):
        S.debug_gemm(A, B, bn=128, out=D)
    torch.cuda.synchronize()
    buf = np.zeros(8, dtype=np.int64)
    lib.seed_debug_gemm_prof(buf.ctypes.data_as(C.c_void_p))
    d = buf - buf[0]
    print(M, N, K, "setup", d[1], "producer issued", d[2], "MMA full", d[3], "MMA committed", d[4],
          "epi start", d[5], "epi end", d[6], "exit", d[7])
