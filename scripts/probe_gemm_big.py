import sys
import torch
sys.path.insert(0, ".")
import paper_1910_06591_b200 as S
M = N = K = 4096
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
D = torch.empty(M, N, device="cuda")
for _ in range(2):
    S.debug_gemm(A, B, bn=256, out=D)
torch.cuda.synchronize()
print("ok")
