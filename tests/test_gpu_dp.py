"""DP equivalence on >= 2 GPUs (H10): an N-rank seed_learner_step with the NCCL
allreduce equals the 1-GPU step on the concatenated batch (fp32 reduction-order
tolerance), and parameters are bit-identical across ranks after Adam."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs 2 GPUs")
@pytest.mark.parametrize("cfg,peer", [("c2", "0"), ("c2", "1"), ("c4", "0")])
def test_dp_two_ranks(tmp_path, cfg, peer):
    """peer=1: the NVLink peer-memory allreduce (seed_comm_peer_*) instead of NCCL;
    c4 = the GRF deep net (BASELINE.json configs[3], the config it scales 1/2/4/8)."""
    n = 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29530 + int(peer) + (10 if cfg == "c4" else 0)),
           os.path.join(ROOT, "scripts", "dp_check.py"), str(tmp_path)]
    subprocess.run(cmd, check=True, timeout=600, env=dict(os.environ, SEED_PEER=peer, CFG=cfg))
    g = [np.load(tmp_path / f"grads{r}.npy") for r in range(n)]
    p = [np.load(tmp_path / f"params{r}.npy") for r in range(n)]
    for r in range(1, n):
        np.testing.assert_array_equal(g[r], g[0])
        np.testing.assert_array_equal(p[r], p[0])      # replicas stay bit-identical
    gf = np.load(tmp_path / "grads_full.npy")
    rel = np.linalg.norm(g[0].astype(np.float64) - gf) / np.linalg.norm(gf)
    assert rel < 1e-4, rel
