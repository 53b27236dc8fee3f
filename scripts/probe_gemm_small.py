import sys
import torch
sys.path.insert(0, ".")
import paper_1910_06591_b200 as S
M, N, K = 268800, 16, 64
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
D = torch.empty(M, N, device="cuda")
for _ in range(3):
    S.debug_gemm(A, B, bn=16, out=D)
torch.cuda.synchronize()
print("ok")
