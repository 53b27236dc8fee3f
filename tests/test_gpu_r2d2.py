"""GPU parity of the R2D2 pieces (include/seed.h
seed_r2d2_targets / seed_replay_*) against the fp64 oracle on the same fp32
inputs.  Tolerances: fp32 arithmetic of a definition -> elementwise
|gpu - ref| <= 1e-5 (|ref| + rms(ref)) (C22's V-trace form); the double-Q argmax,
slots, generations and payload bytes are integer / byte work -> exact (sampled
slots exact except draws within 1e-5 of a CDF boundary, where fp32 and fp64 may
legitimately disagree — C18's rule)."""
import math

import numpy as np
import pytest
import torch

import oracle as O
import seedgen

pytestmark = pytest.mark.gpu


def _S():
    import paper_1910_06591_b200 as S
    return S


def _scaled(gpu, ref, tol=1e-5, what=""):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = math.sqrt(float(np.mean(ref ** 2))) if ref.size else 0.0
    err = np.abs(gpu - ref)
    bound = tol * (np.abs(ref) + rms) + 1e-30
    assert np.all(err <= bound), f"{what}: worst {np.max(err / bound):.3g}"


def _case(B, T, A, seed, done_p=0.05):
    g = seedgen.rng(seed)
    f = np.float32
    qo = g.normal(0, 2.0, (B, T + 1, A)).astype(f)
    qt = g.normal(0, 2.0, (B, T + 1, A)).astype(f)
    a = g.integers(0, A, (B, T + 1)).astype(np.int32)
    r = (g.normal(0, 1, (B, T)) * (g.random((B, T)) < 0.3)).astype(f)
    disc = (0.997 * (g.random((B, T)) >= done_p)).astype(f)
    w = g.uniform(0.2, 1.0, B).astype(f)
    return qo, qt, a, r, disc, w


@pytest.mark.parametrize("B,T,A,n", [(1, 1, 2, 5), (3, 7, 4, 5), (64, 80, 18, 5), (33, 120, 18, 1),
                                     (17, 40, 9, 3), (5, 31, 32, 7)])
def test_r2d2_targets_parity(B, T, A, n):
    S = _S()
    qo, qt, a, r, disc, w = _case(B, T, A, seed=B * 100 + T)
    d = {k: torch.from_numpy(v).cuda() for k, v in dict(qo=qo, qt=qt, a=a, r=r, disc=disc, w=w).items()}
    y, delta, prio, dq, loss = S.r2d2_targets(d["qo"], d["qt"], d["a"], d["r"], d["disc"], n=n,
                                              eta=0.9, is_weights=d["w"], loss_scale=1.0 / (B * T),
                                              want_grad=True)
    torch.cuda.synchronize()
    ry, rd, rp = O.r2d2_targets(qo, qt, a, r, disc, n=n, eta=0.9)
    _scaled(y.cpu().numpy(), ry, what="y")
    _scaled(delta.cpu().numpy(), rd, what="delta")
    _scaled(prio.cpu().numpy(), rp, what="priority")
    rl, rdq = O.r2d2_loss_grad(qo, a, ry, w, 1.0 / (B * T))
    _scaled(dq.cpu().numpy(), rdq, what="dq")
    _scaled(loss.cpu().numpy().sum(), rl, 1e-4, what="loss")


def test_r2d2_targets_goldens_on_gpu():
    """terminal step with r = 1 -> y = rescale(1) = 0.41521 (fp32)."""
    S = _S()
    z = torch.zeros(1, 2, 3, device="cuda")
    y, _, _, _, _ = S.r2d2_targets(z, torch.full_like(z, 7.0), torch.zeros(1, 2, dtype=torch.int32,
                                                                           device="cuda"),
                                   torch.ones(1, 1, device="cuda"), torch.zeros(1, 1, device="cuda"))
    assert abs(float(y.item()) - 0.41521356237309515) < 1e-6


def _replay(slots, alpha=0.9, beta=0.6, rb=64):
    S = _S()
    return S.PrioritizedReplay(slots, rb, alpha, beta)


def test_replay_insert_update_sample_parity():
    R = _replay(300)
    g = seedgen.rng(7)
    rec = torch.from_numpy(g.integers(0, 256, (300, 64), dtype=np.uint8)).cuda()
    slots, gens = R.insert(rec)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(slots.cpu().numpy(), np.arange(300))
    np.testing.assert_array_equal(gens.cpu().numpy(), 1)
    assert torch.equal(R.data, rec)                       # payload scatter, bit-exact
    np.testing.assert_allclose(R.tree[R.capacity:R.capacity + 300].cpu().numpy(), 1.0)
    pr = (g.random(300) * 4).astype(np.float32)
    pr[7] = 0.0
    R.update(slots, gens, torch.from_numpy(pr).cuda())
    torch.cuda.synchronize()
    tree = R.tree.cpu().numpy().astype(np.float64)
    leaves = tree[R.capacity:R.capacity + 300]
    _scaled(leaves, pr.astype(np.float64) ** 0.9, 1e-6, "leaves = p^alpha")
    # every internal node = left + right (fp32, exact per pairwise add) and the root
    C = R.capacity
    for k in range(1, C):
        assert tree[k] == np.float32(np.float32(tree[2 * k]) + np.float32(tree[2 * k + 1]))
    assert abs(tree[1] - (pr.astype(np.float64) ** 0.9).sum()) <= 1e-5 * tree[1]
    assert abs(float(R.max_priority.item()) - pr.max()) == 0
    u = g.random(512).astype(np.float32)
    s_gpu, gen_gpu, w_gpu = R.sample(512, uniforms=torch.from_numpy(u).cuda())
    torch.cuda.synchronize()
    ri, rw = O.replay_sample(pr, u, 0.9, 0.6, size=300)
    s_gpu = s_gpu.cpu().numpy()
    c = np.cumsum(pr.astype(np.float64) ** 0.9)
    near = np.min(np.abs(c[None, :] - (u.astype(np.float64) * c[-1])[:, None]), axis=1) < 1e-5 * c[-1]
    assert np.all((s_gpu == ri) | near), np.nonzero((s_gpu != ri) & ~near)
    assert np.all(pr[s_gpu] > 0)                            # a zero priority is never drawn
    ok = s_gpu == ri
    _scaled(w_gpu.cpu().numpy()[ok], rw[ok], 1e-4, "importance weights")
    np.testing.assert_array_equal(gen_gpu.cpu().numpy(), 1)
    # gather: the sampled sequences' payload, bit-exact
    out = R.gather(torch.from_numpy(s_gpu).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), rec.cpu().numpy()[s_gpu])


def test_replay_fifo_eviction_and_stale_updates():
    """FIFO eviction at capacity, new sequences at the max priority seen, and an update
    carrying an evicted sequence's generation is skipped."""
    R = _replay(8)
    rec = torch.zeros(8, 64, dtype=torch.uint8, device="cuda")
    s1, g1 = R.insert(rec)
    R.update(s1, g1, torch.arange(1, 9, dtype=torch.float32, device="cuda"))
    s2, g2 = R.insert(rec[:3])                              # evicts slots 0..2
    torch.cuda.synchronize()
    np.testing.assert_array_equal(s2.cpu().numpy(), [0, 1, 2])
    np.testing.assert_array_equal(g2.cpu().numpy(), [2, 2, 2])
    leaves = R.tree[R.capacity:R.capacity + 8].cpu().numpy()
    np.testing.assert_allclose(leaves[:3], 8.0 ** 0.9, rtol=1e-6)     # max priority seen
    # stale update (generation 1) for slot 1 is skipped; a current one is applied
    R.update(torch.tensor([1, 2], dtype=torch.int32, device="cuda"),
             torch.tensor([1, 2], dtype=torch.int32, device="cuda"),
             torch.tensor([0.5, 0.25], device="cuda"))
    torch.cuda.synchronize()
    leaves = R.tree[R.capacity:R.capacity + 8].cpu().numpy()
    np.testing.assert_allclose(leaves[1], 8.0 ** 0.9, rtol=1e-6)
    np.testing.assert_allclose(leaves[2], 0.25 ** 0.9, rtol=1e-6)
    assert R.size.cpu().numpy().tolist()[:3] == [8, 3, 0]
    # invalid priorities are rejected and counted
    R.update(torch.tensor([3], dtype=torch.int32, device="cuda"),
             torch.tensor([1], dtype=torch.int32, device="cuda"),
             torch.tensor([float("nan")], device="cuda"))
    torch.cuda.synchronize()
    assert int(R.size[2].item()) == 1


def test_replay_sampling_distribution_philox():
    """Device Philox draws over a 2^17-leaf tree (the paper's 10^5 sequences):
    a chi-square goodness-of-fit against p^alpha / sum over coarse bins."""
    n = 100000
    R = _replay(n, rb=16)
    g = seedgen.rng(9)
    s, gg = R.insert(torch.zeros(1024, 16, dtype=torch.uint8, device="cuda"))
    for _ in range(n // 1024 - 1):
        R.insert(torch.zeros(1024, 16, dtype=torch.uint8, device="cuda"))
    R.insert(torch.zeros(n % 1024, 16, dtype=torch.uint8, device="cuda"))
    pr = g.random(n).astype(np.float32) * 3
    slots = torch.arange(n, dtype=torch.int32, device="cuda")
    for k in range(0, n, 1024):
        R.update(slots[k:k + 1024], torch.ones(min(1024, n - k), dtype=torch.int32, device="cuda"),
                 torch.from_numpy(pr[k:k + 1024]).cuda())
    counts = np.zeros(n, np.int64)
    for c in range(200):
        sl, _, w = R.sample(1024, seed=11, counter=c)
        counts += np.bincount(sl.cpu().numpy(), minlength=n)
    torch.cuda.synchronize()
    P = O.replay_probabilities(pr, 0.9)
    bins = np.arange(n) // 1000                          # 100 bins of 1000 sequences
    obs = np.bincount(bins, weights=counts)
    exp = np.bincount(bins, weights=P) * counts.sum()
    from scipy.stats import chisquare
    assert chisquare(obs, exp).pvalue > 1e-3


def _r2d2_step_case(cfg, B, bi, T, seed):
    S = _S()
    spec = S.spec_for_config(cfg)
    ospec = {"c2": O.spec_c2, "c4": O.spec_c4}[cfg]()
    layout = O.param_layout(ospec)
    params = seedgen.glorot_params(layout, seed=seed, bias_std=0.1)
    tparams = seedgen.glorot_params(layout, seed=seed + 1, bias_std=0.1)
    full = seedgen.learner_batch((ospec.obs_h, ospec.obs_w, ospec.obs_c), ospec.num_actions, B,
                                 bi + T, seed=seed + 2, done_p=0.08, smm=(cfg == "c4"))
    L1 = bi + T + 1
    burn = {k: np.ascontiguousarray(v[:, :bi]) if v.ndim >= 2 and v.shape[1] == L1 else v
            for k, v in full.items()}
    train = {k: np.ascontiguousarray(v[:, bi:]) if v.ndim >= 2 and v.shape[1] == L1 else v
             for k, v in full.items()}
    w = seedgen.rng(seed + 3).uniform(0.3, 1.0, B).astype(np.float32)
    hp = S.R2d2HParams(n=3, loss_scale=1.0 / (B * T), lr=1e-4)
    return S, spec, ospec, params, tparams, burn, train, w, hp


@pytest.mark.parametrize("cfg,B,bi,T", [("c2", 3, 4, 5), ("c2", 2, 0, 6), ("c4", 2, 2, 3)])
def test_r2d2_learner_step_parity(cfg, B, bi, T):
    """seed_r2d2_learner_step (burn-in, online / target forward, dueling heads, n-step
    double-Q targets, IS-weighted backward, clip 80 + Adam) against the oracle:
    Q values and priorities at C22 vs the bf16-emulated oracle, every gradient tensor
    at C22 vs emulated and within C31's bound of the exact definition, the Adam update
    and the version counter."""
    S, spec, ospec, params, tparams, burn, train, w, hp = _r2d2_step_case(cfg, B, bi, T, 11)
    Lr = S.R2d2Learner(spec, bi, T, B, params, hp)
    Lr.target_params.copy_(torch.from_numpy(tparams))
    Lr.target_lowp.copy_(_lowp_of(S, spec, tparams))
    gb = lambda d: {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in d.items()}
    m, prio = Lr.step(gb(train), burn=gb(burn) if bi > 0 else None,
                      is_weights=torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    hpo = dict(discount=float(np.float32(hp.discount)), n=hp.n, eta=float(np.float32(hp.eta)),
               rescale_eps=float(np.float32(hp.rescale_eps)), loss_scale=float(np.float32(hp.loss_scale)),
               lr=float(np.float32(hp.lr)), beta1=float(np.float32(hp.beta1)),
               beta2=float(np.float32(hp.beta2)), eps=float(np.float32(hp.eps)),
               max_grad_norm=float(np.float32(hp.max_grad_norm)))
    z = np.zeros(params.size)
    bo = burn if bi > 0 else None
    emu = O.r2d2_learner_step(ospec, params, tparams, z, z, 0, bo, train, w, hpo, emu=True)
    ex = O.r2d2_learner_step(ospec, params, tparams, z, z, 0, bo, train, w, hpo)
    from test_gpu_learner import bf16_check, exact_bound_check
    bf16_check(prio.cpu().numpy(), emu["priorities"], "priorities vs emulated")
    exact_bound_check(prio.cpu().numpy(), ex["priorities"], emu["priorities"], "priorities vs exact")
    g = Lr.grads.cpu().numpy().astype(np.float64)
    gt, gr, gx = O.unflatten(ospec, g), O.unflatten(ospec, emu["grads"]), O.unflatten(ospec, ex["grads"])
    deep = cfg != "c2"
    if deep:   # C31's deep-torso rule: the whole gradient within 1.25x, each tensor 1.5x
        allg = np.concatenate([np.ravel(gt[n]) for n in gt])
        exact_bound_check(allg, np.concatenate([np.ravel(gx[n]) for n in gt]),
                          np.concatenate([np.ravel(gr[n]) for n in gt]), "whole gradient vs exact")
    for n, _ in O.param_layout(ospec):
        # C22 vs the emulated oracle for the whole Atari net and for the deep nets' core
        # and heads; the deep torso / FC gradients sit below 15-20 bf16 convs whose mask
        # flips make the emulated oracle a sampling comparison there (C30 / C31)
        if not deep or n.startswith(("lstm", "heads")):
            bf16_check(gt[n], gr[n], f"grad {n} vs emulated")
        exact_bound_check(gt[n], gx[n], gr[n], f"grad {n} vs exact", factor=1.5 if deep else 1.25)
    mm = m.cpu().numpy()
    assert mm[5] == 1.0 and int(Lr.step_counter.item()) == 1
    assert abs(mm[0] - emu["loss"]) <= 2e-2 * abs(emu["loss"])
    _scaled(mm[4], emu["grad_norm"], 2e-2, "grad norm")
    # clip (80) + Adam on the GPU's own gradients (Adam normalises every coordinate, so
    # the update is compared on identical inputs, as in the V-trace learner tests)
    p2, m2, v2, step2, norm, applied = O.clip_adam(params.astype(np.float64), g, np.zeros(params.size),
                                                   np.zeros(params.size), 0, hpo)
    assert applied == 1
    _scaled(mm[4], norm, 1e-5, "grad norm (own grads)")
    _scaled(Lr.m.cpu().numpy(), m2, 1e-5, "adam m")
    _scaled(Lr.v.cpu().numpy(), v2, 1e-5, "adam v")
    # the update against the fp32 rounding of the stored parameter: with the R2D2 Adam
    # epsilon (1e-3) the per-coordinate updates can be ~1e-8, a few fp32 ulps of p
    d_gpu = Lr.params.cpu().numpy().astype(np.float64) - params
    d_ref = p2 - params
    bound = 1e-3 * (np.abs(d_ref) + np.sqrt(np.mean(d_ref ** 2))) + 2 * np.abs(params) * 2.0 ** -23
    assert np.all(np.abs(d_gpu - d_ref) <= bound), np.max(np.abs(d_gpu - d_ref) / bound)


def _lowp_of(S, spec, params):
    """The bf16 operand image of a parameter vector (seed_net_refresh_lowp)."""
    L = S.Learner(spec, 1, 1, params)
    return L.lowp.clone()
