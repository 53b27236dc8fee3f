"""GPU parity of seed_vtrace (K1) against the fp64 oracle (tolerance C22:
|gpu - ref| <= 1e-5 (|ref| + rms(ref)) elementwise)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import seedgen

pytestmark = pytest.mark.gpu


def _tol_check(gpu, ref, tol=1e-5):
    gpu = np.asarray(gpu, np.float64)
    rms = math.sqrt(float(np.mean(ref ** 2))) if ref.size else 0.0
    err = np.abs(gpu - ref)
    bound = tol * (np.abs(ref) + rms)
    bad = err > bound
    assert not bad.any(), f"{bad.sum()} elems out of tol; worst {np.max(err / (bound + 1e-30)):.3g}"


def _run(x, rho_bar, c_bar, lam):
    import paper_1910_06591_b200 as S
    d = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in x.items()}
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    vs, pg = S.vtrace(d["behaviour_logp"], d["target_logp"], d["rewards"], d["discounts"],
                      d["values"], d["bootstrap"], rho_bar, c_bar, lam, nonfinite_flag=flag)
    torch.cuda.synchronize()
    return vs.cpu().numpy(), pg.cpu().numpy(), int(flag.item())


CASES = [(1, 1), (3, 5), (4, 9), (20, 8), (20, 1000), (32, 77), (100, 33), (128, 10),
         (130, 17), (257, 5), (99, 64)]


@pytest.mark.parametrize("T,B", CASES)
@pytest.mark.parametrize("clip", [(1.0, 1.0, 1.0), (1.0, 1.0, 0.95), (2.0, 0.5, 0.9),
                                  (math.inf, math.inf, 1.0)])
def test_vtrace_parity(T, B, clip):
    rb, cb, lam = clip
    for seed in (0, 1, 2):
        x = seedgen.vtrace_inputs(B, T, seed=seed, done_p=0.05)
        vs_r, pg_r, bad = O.vtrace(**x, rho_bar=rb, c_bar=cb, lam=lam)
        vs, pg, flag = _run(x, rb, cb, lam)
        _tol_check(vs, vs_r)
        _tol_check(pg, pg_r)
        assert flag == int(bad) == 0


@pytest.mark.parametrize("edge", ["done0", "doneLast", "alldone", "nodone", "onpolicy"])
def test_vtrace_edges(edge):
    T, B = 37, 50
    x = seedgen.vtrace_inputs(B, T, seed=5, done_p=0.0 if edge == "nodone" else 0.05)
    if edge == "done0":
        x["discounts"][:, 0] = 0
    if edge == "doneLast":
        x["discounts"][:, T - 1] = 0
    if edge == "alldone":
        x["discounts"][:] = 0
    if edge == "onpolicy":
        x["target_logp"] = x["behaviour_logp"].copy()   # ratio exactly 1
    vs_r, pg_r, _ = O.vtrace(**x, rho_bar=1.0, c_bar=1.0, lam=0.99)
    vs, pg, _ = _run(x, 1.0, 1.0, 0.99)
    _tol_check(vs, vs_r)
    _tol_check(pg, pg_r)


def test_vtrace_nonfinite_flag():
    x = seedgen.vtrace_inputs(9, 12, seed=1)
    x["target_logp"][4, 7] = np.nan
    _, _, flag = _run(x, 1.0, 1.0, 1.0)
    assert flag == 1


def test_vtrace_full_size_sampled():
    """bench shape T=100, B=2^17: oracle on a sample of 2048 trajectories."""
    T, B = 100, 1 << 17
    x = seedgen.vtrace_inputs(B, T, seed=0)
    vs, pg, flag = _run(x, 1.0, 1.0, 1.0)
    idx = seedgen.rng(1).choice(B, 2048, replace=False)
    sub = {k: v[idx] for k, v in x.items()}
    vs_r, pg_r, _ = O.vtrace(**sub, rho_bar=1.0, c_bar=1.0, lam=1.0)
    _tol_check(vs[idx], vs_r)
    _tol_check(pg[idx], pg_r)
    assert flag == 0


@pytest.mark.parametrize("name", ["vtrace_S145.json", "vtrace_cbar_hand.json"])
def test_vtrace_golden_values(name):
    """The kernel on the printed / hand-derived examples (tests/golden): values fixed by
    the paper's recursion, not by the oracle (fp32 inputs: 1e-5 relative)."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", name)) as f:
        g = json.load(f)
    x = {k: np.asarray(g[k], np.float32) for k in ("behaviour_logp", "target_logp", "rewards",
                                                   "discounts", "values", "bootstrap")}
    vs, pg, flag = _run(x, g["rho_bar"], g["c_bar"], g["lambda"])
    _tol_check(vs, np.asarray(g["vs"], np.float64))
    _tol_check(pg, np.asarray(g["pg_advantages"], np.float64))
    assert flag == 0
