"""tcgen05 GEMM engine (seed_debug_gemm) vs an fp64 CPU product of the same bf16
operands: all operand-major combinations, every BN tile, split-K, ragged M/N/K."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bn", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("at,bt", [(False, False), (False, True), (True, False), (True, True)])
@pytest.mark.parametrize("M,N,K,splits", [(128, 64, 64, 1), (200, 40, 136, 1),
                                          (384, 256, 1024, 1), (256, 32, 4096, 5),
                                          (200, 40, 136, -1), (256, 32, 4096, -3),
                                          (1152, 48, 520, 1)])
def test_gemm_engine(bn, at, bt, M, N, K, splits):
    import paper_1910_06591_b200 as S
    g = torch.Generator().manual_seed(M * 7 + N * 3 + K)
    A = torch.randn(M, K, generator=g).to(torch.bfloat16)
    B = torch.randn(N, K, generator=g).to(torch.bfloat16)
    ref = A.double() @ B.double().T
    Ad = (A.T.contiguous() if at else A).cuda()
    Bd = (B.T.contiguous() if bt else B).cuda()
    D = S.debug_gemm(Ad, Bd, a_t=at, b_t=bt, bn=bn, splits=splits)
    torch.cuda.synchronize()
    err = (D.cpu().double() - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
