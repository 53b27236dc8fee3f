"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a worked example printed in
SPEC.md (golden files under tests/golden/), a closed form, exact enumeration,
finite differences, or an independent library routine (torch CPU fp64).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O
import seedgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ V-trace
def test_vtrace_worked_example_S145():
    g = _gold("vtrace_S145.json")
    vs, pg, bad = O.vtrace(g["behaviour_logp"], g["target_logp"], g["rewards"], g["discounts"],
                           g["values"], g["bootstrap"], g["rho_bar"], g["c_bar"], g["lambda"])
    np.testing.assert_allclose(vs, g["vs"], atol=1e-12)
    np.testing.assert_allclose(pg, g["pg_advantages"], atol=1e-12)
    assert not bad


def test_vtrace_cbar_lambda_hand_golden():
    """c_bar and lambda pinned by a hand-derived example (tests/golden/vtrace_cbar_hand.json,
    S:140 with rho_bar != c_bar and lambda < 1): the direct sum repeats the recursion's
    formula for c_t, and the enumeration / lambda-return pins are blind to c_bar."""
    g = _gold("vtrace_cbar_hand.json")
    vs, pg, bad = O.vtrace(g["behaviour_logp"], g["target_logp"], g["rewards"], g["discounts"],
                           g["values"], g["bootstrap"], g["rho_bar"], g["c_bar"], g["lambda"])
    np.testing.assert_allclose(vs, g["vs"], atol=1e-9)
    np.testing.assert_allclose(pg, g["pg_advantages"], atol=1e-9)
    assert not bad


def test_vtrace_monotone_clipping_S161():
    """with rho_bar' <= rho_bar and identical inputs, the outputs differ only
    through the clipped ratios.  Pre-clipping every ratio to rho_bar' (target log-prob
    rewritten as log mu + log min(ratio, rho_bar')) and running with rho_bar must give
    exactly the rho_bar' result: rho' = min(rho_bar, ratio') = min(ratio, rho_bar') and,
    for c_bar <= rho_bar', c' = lambda min(c_bar, ratio') = lambda min(c_bar, ratio)."""
    x = seedgen.vtrace_inputs(16, 24, seed=17)
    blp = x["behaviour_logp"].astype(np.float64)
    tlp = blp + 1.2 * seedgen.rng(18).standard_normal(blp.shape)   # ratios well above / below 1
    for rb, rb2, cb, lam in ((2.0, 1.0, 1.0, 0.95), (np.inf, 1.5, 0.7, 0.9), (3.0, 0.8, 0.5, 1.0)):
        base = dict(rewards=x["rewards"], discounts=x["discounts"], values=x["values"],
                    bootstrap=x["bootstrap"])
        vs2, pg2, _ = O.vtrace(blp, tlp, **base, rho_bar=rb2, c_bar=cb, lam=lam)
        ratio = np.exp(tlp - blp)
        tlp_c = blp + np.log(np.minimum(ratio, rb2))
        vs1, pg1, _ = O.vtrace(blp, tlp_c, **base, rho_bar=rb, c_bar=cb, lam=lam)
        np.testing.assert_allclose(vs1, vs2, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(pg1, pg2, rtol=1e-12, atol=1e-12)
        # and the looser clip really differs where some ratio exceeds rho_bar'
        vs0, _, _ = O.vtrace(blp, tlp, **base, rho_bar=rb, c_bar=cb, lam=lam)
        assert np.max(np.abs(vs0 - vs2)) > 1e-3


def test_vtrace_fully_clipped_S146():
    x = seedgen.vtrace_inputs(4, 7, seed=3)
    tlp = x["behaviour_logp"] - 1e4            # ratio underflows to 0 -> rho = c = 0
    vs, pg, _ = O.vtrace(x["behaviour_logp"], tlp, x["rewards"], x["discounts"], x["values"],
                         x["bootstrap"], 1.0, 1.0, 1.0)
    np.testing.assert_array_equal(vs, x["values"].astype(np.float64))
    np.testing.assert_array_equal(pg, 0.0)


def test_vtrace_done_at_zero_S147():
    x = seedgen.vtrace_inputs(5, 6, seed=4, force_done_at=0)
    vs, _, _ = O.vtrace(x["behaviour_logp"], x["target_logp"], x["rewards"], x["discounts"],
                        x["values"], x["bootstrap"], 1.0, 1.0, 0.95)
    rho0 = np.minimum(1.0, np.exp(x["target_logp"][:, 0].astype(np.float64)
                                  - x["behaviour_logp"][:, 0]))
    V0 = x["values"][:, 0].astype(np.float64)
    np.testing.assert_allclose(vs[:, 0], V0 + rho0 * (x["rewards"][:, 0] - V0), atol=1e-12)


def _lambda_return_forward(r, g, V, boot, lam):
    """Forward-accumulated lambda-return (Sutton & Barto): G^lam_s =
    (1-lam) sum_{n=1}^{N-1} lam^{n-1} G^(n)_s + lam^{N-1} G^(N)_s, per-step gammas."""
    B, T = V.shape
    Vx = np.concatenate([V, boot[:, None]], axis=1)
    out = np.zeros((B, T))
    for s in range(T):
        N = T - s
        total = np.zeros(B)
        for n in range(1, N + 1):
            Gn = np.zeros(B)
            disc = np.ones(B)
            for k in range(n):
                Gn += disc * r[:, s + k]
                disc = disc * g[:, s + k]
            Gn += disc * Vx[:, s + n]
            w = (1 - lam) * lam ** (n - 1) if n < N else lam ** (N - 1)
            total += w * Gn
        out[:, s] = total
    return out


@pytest.mark.parametrize("lam", [0.9, 0.95, 0.99, 1.0])
def test_vtrace_onpolicy_is_lambda_return(lam):
    """north_star pin: pi = mu, no clip active -> vs = lambda-weighted n-step target."""
    for seed in range(20):
        T = 1 + seed % 10
        x = seedgen.vtrace_inputs(6, T, seed=seed, done_p=0.15)
        vs, pg, _ = O.vtrace(x["behaviour_logp"], x["behaviour_logp"], x["rewards"],
                             x["discounts"], x["values"], x["bootstrap"], 1.0, 1.0, lam)
        ref = _lambda_return_forward(x["rewards"].astype(np.float64),
                                     x["discounts"].astype(np.float64),
                                     x["values"].astype(np.float64),
                                     x["bootstrap"].astype(np.float64), lam)
        np.testing.assert_allclose(vs, ref, rtol=1e-11, atol=1e-11)
        if lam == 1.0:   # identity: on-policy lambda=1 -> pg_adv = vs - V
            np.testing.assert_allclose(pg, vs - x["values"], atol=1e-11)


def test_vtrace_direct_sum_equals_recursion():
    for seed in range(30):
        T = 1 + seed % 8
        x = seedgen.vtrace_inputs(3, T, seed=100 + seed, done_p=0.2)
        rb, cb, lam = [(np.inf, 1.0, 1.0), (1.0, 1.0, 0.9), (2.0, 0.5, 0.95)][seed % 3]
        a = O.vtrace(**x, rho_bar=rb, c_bar=cb, lam=lam)
        b = O.vtrace_direct(**x, rho_bar=rb, c_bar=cb, lam=lam)
        np.testing.assert_allclose(a[0], b[0], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(a[1], b[1], rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("rho_bar,c_bar,lam", [(np.inf, 1.0, 1.0), (1.0, 1.0, 1.0),
                                               (0.7, 0.5, 0.9), (2.0, 1.0, 0.95)])
def test_vtrace_exact_enumeration_fixed_point(rho_bar, c_bar, lam):
    """IMPALA Thm. 1 (cited at P:145): with V = V^{pi_rho}, the value of
    pi_rho(a|x) ~ min(rho_bar mu(a|x), pi(a|x)), E_mu[v_0] = V(x_0) exactly.
    Exact expectation by enumerating all 2^T action x 3^T next-state sequences."""
    g = seedgen.rng(7)
    S, A, T, gamma = 3, 2, 3, 0.9
    mu = g.dirichlet(np.ones(A), size=S)
    pi = g.dirichlet(np.ones(A), size=S)
    P = g.dirichlet(np.ones(S), size=(S, A))
    R = g.standard_normal((S, A))
    prho = np.minimum(rho_bar * mu, pi)
    prho = prho / prho.sum(axis=1, keepdims=True)
    # V^{pi_rho}: solve (I - gamma P_pi) V = r_pi
    Ppi = np.einsum("sa,sat->st", prho, P)
    rpi = (prho * R).sum(axis=1)
    Vst = np.linalg.solve(np.eye(S) - gamma * Ppi, rpi)
    for x0 in range(S):
        expect = 0.0
        for acts in itertools.product(range(A), repeat=T):
            for nxt in itertools.product(range(S), repeat=T):
                xs = [x0] + list(nxt)
                prob = 1.0
                for t in range(T):
                    prob *= mu[xs[t], acts[t]] * P[xs[t], acts[t], xs[t + 1]]
                blp = np.log([[mu[xs[t], acts[t]] for t in range(T)]])
                tlp = np.log([[pi[xs[t], acts[t]] for t in range(T)]])
                r = np.array([[R[xs[t], acts[t]] for t in range(T)]])
                V = np.array([[Vst[xs[t]] for t in range(T)]])
                vs, _, _ = O.vtrace(blp, tlp, r, np.full((1, T), gamma), V,
                                    np.array([Vst[xs[T]]]), rho_bar, c_bar, lam)
                expect += prob * vs[0, 0]
        assert abs(expect - Vst[x0]) < 1e-12, (x0, expect, Vst[x0])


def test_vtrace_episode_isolation_S162():
    x = seedgen.vtrace_inputs(4, 12, seed=9, done_p=0.0)
    x["discounts"][:, 5] = 0.0                       # episode boundary after step 5
    vs1, _, _ = O.vtrace(**x, rho_bar=1.0, c_bar=1.0, lam=0.95)
    y = {k: v.copy() for k, v in x.items()}
    y["rewards"][:, 6:] += 5.0
    y["values"][:, 6:] -= 2.0
    vs2, _, _ = O.vtrace(**y, rho_bar=1.0, c_bar=1.0, lam=0.95)
    np.testing.assert_array_equal(vs1[:, :6], vs2[:, :6])


def test_vtrace_nonfinite_flag_S143():
    x = seedgen.vtrace_inputs(2, 4, seed=1)
    x["target_logp"][1, 2] = np.nan
    assert O.vtrace(**x)[2]
    x = seedgen.vtrace_inputs(2, 4, seed=1)
    assert not O.vtrace(**x)[2]


# ------------------------------------------------------------------ loss
HP = dict(discount=0.99, rho_bar=1.0, c_bar=1.0, **{"lambda": 0.95}, vf_coef=0.5,
          ent_coef=0.01, loss_scale=1.0, lr=3e-4, beta1=0.9, beta2=0.999, eps=1e-5,
          max_grad_norm=40.0)


def test_loss_closed_forms_S155_S157():
    gold = _gold("loss_S155_157.json")
    # (b) single step (T=1 plus bootstrap slot), 2 actions, logits [0,0], action 0,
    # pg_adv = 1, v = V: make r + g*v_T - V = 1 with rho = 1 and vs = V via c = 0 ... use
    # the definition directly: values V_0 = 0, bootstrap 0, reward 1, discount 0.
    logits = np.zeros((1, 2, 2))
    values = np.zeros((1, 2))
    act = np.zeros((1, 2), np.int32)
    blp = np.full((1, 2), math.log(0.5))
    rew = np.array([[0.0, 1.0]])
    done = np.array([[0, 1]])
    hp = dict(HP, ent_coef=0.0, vf_coef=0.0, discount=0.9)
    L = O.policy_loss(logits, values, act, blp, rew, done, hp)
    assert L["pg_adv"][0, 0] == pytest.approx(1.0)
    assert L["pg"] == pytest.approx(gold["pg_term_b"], abs=1e-12)
    # (c) entropy of a uniform 4-action policy
    logits4 = np.zeros((1, 2, 4))
    L4 = O.policy_loss(logits4, values, act, np.full((1, 2), math.log(0.25)),
                       np.zeros((1, 2)), np.zeros((1, 2)), dict(HP, ent_coef=0.01))
    assert L4["entropy_t"][0, 0] == pytest.approx(gold["entropy_uniform4"], abs=1e-12)
    assert L4["entropy"] == pytest.approx(gold["entropy_term_c"], abs=1e-12)
    # (a) ent_coef = 0, uniform logits, pg_adv = 0 (zero rewards, values 0) -> loss 0
    L0 = O.policy_loss(logits4, values, act, np.full((1, 2), math.log(0.25)),
                       np.zeros((1, 2)), np.zeros((1, 2)), dict(HP, ent_coef=0.0))
    assert L0["loss"] == 0.0


def test_loss_gradients_vs_torch_autograd():
    """dlogits/dvalues vs torch autograd of the S:152 loss with the V-trace
    targets held constant (stop-gradient)."""
    g = seedgen.rng(5)
    B, T, A = 3, 6, 5
    logits = g.standard_normal((B, T + 1, A))
    values = g.standard_normal((B, T + 1))
    act = g.integers(0, A, (B, T + 1))
    blp = -np.log(A) + 0.3 * g.standard_normal((B, T + 1))
    rew = g.standard_normal((B, T + 1))
    done = (g.random((B, T + 1)) < 0.2).astype(np.uint8)
    hp = dict(HP, loss_scale=1.0 / (B * T), ent_coef=0.03)
    L = O.policy_loss(logits, values, act, blp, rew, done, hp)
    z = torch.tensor(logits, dtype=torch.float64, requires_grad=True)
    v = torch.tensor(values, dtype=torch.float64, requires_grad=True)
    logp = torch.log_softmax(z[:, :T], dim=-1)
    tl = logp.gather(2, torch.tensor(act[:, :T])[:, :, None])[:, :, 0]
    ent = -(logp.exp() * logp).sum(-1)
    vs = torch.tensor(L["vs"])
    pg = torch.tensor(L["pg_adv"])
    s = hp["loss_scale"]
    loss = s * ((-pg * tl).sum() + 0.5 * hp["vf_coef"] * ((vs - v[:, :T]) ** 2).sum()
                - hp["ent_coef"] * ent.sum())
    loss.backward()
    assert float(loss.detach()) == pytest.approx(L["loss"], rel=1e-12)
    np.testing.assert_allclose(L["dlogits"], z.grad.numpy(), atol=1e-13)
    np.testing.assert_allclose(L["dvalues"], v.grad.numpy(), atol=1e-13)
    # invariant: softmax gradients sum to zero per (b,t)
    np.testing.assert_allclose(L["dlogits"].sum(-1), 0.0, atol=1e-14)


# ------------------------------------------------------------------ network
def _torch_net(spec, flat, batch):
    """Independent torch CPU fp64 model of the C14/C15 architecture built from
    library routines (conv2d, max_pool2d, LSTMCell)."""
    P = {}
    off = 0
    for name, shape in O.param_layout(spec):
        n = int(np.prod(shape))
        P[name] = torch.tensor(np.asarray(flat[off:off + n], np.float64).reshape(shape),
                               requires_grad=True)
        off += n
    obs = batch["obs"]
    B, T1 = obs.shape[:2]
    A = spec.num_actions
    if spec.kind == O.NET_MLP:
        x = torch.tensor(obs.reshape(B * T1, -1), dtype=torch.float64)
        for i in range(len(spec.mlp_hidden)):
            x = F.relu(F.linear(x, P[f"mlp{i}.w"], P[f"mlp{i}.b"]))
        hfeat = x
    else:
        x = torch.tensor(obs.reshape((B * T1,) + obs.shape[2:]), dtype=torch.float64) / 255.0
        x = x.permute(0, 3, 1, 2)
        cw = lambda n: P[n].permute(0, 3, 1, 2)
        if spec.kind == O.NET_ATARI_SHALLOW:
            x = F.relu(F.conv2d(x, cw("conv1.w"), P["conv1.b"], stride=4))
            x = F.relu(F.conv2d(x, cw("conv2.w"), P["conv2.b"], stride=2))
        else:
            for s in range(len(spec.sections)):
                x = F.conv2d(x, cw(f"s{s}.conv.w"), P[f"s{s}.conv.b"], padding=1)
                H, W = x.shape[2:]
                ph = max((-(-H // 2) - 1) * 2 + 3 - H, 0)
                pw = max((-(-W // 2) - 1) * 2 + 3 - W, 0)
                x = F.pad(x, (pw // 2, pw - pw // 2, ph // 2, ph - ph // 2), value=-math.inf)
                x = F.max_pool2d(x, 3, 2)
                for r in range(2):
                    t = F.conv2d(F.relu(x), cw(f"s{s}.res{r}.conv0.w"), P[f"s{s}.res{r}.conv0.b"],
                                 padding=1)
                    t = F.conv2d(F.relu(t), cw(f"s{s}.res{r}.conv1.w"), P[f"s{s}.res{r}.conv1.b"],
                                 padding=1)
                    x = x + t
            x = F.relu(x)
        flat_x = x.permute(0, 2, 3, 1).reshape(B * T1, -1)
        fc = F.relu(F.linear(flat_x, P["fc.w"], P["fc.b"]))
        done = torch.tensor(batch["done"].astype(bool))
        pa = torch.tensor(batch["prev_action"].astype(np.int64)).reshape(-1)
        oh = F.one_hot(pa.clamp(min=0), A).double() * (pa >= 0)[:, None]
        oh = oh * (~done.reshape(-1))[:, None]
        r = torch.tensor(batch["reward"], dtype=torch.float64).reshape(-1).clamp(-1, 1)
        r = r * (~done.reshape(-1))
        X = torch.cat([fc, oh, r[:, None]], 1).reshape(B, T1, -1)
        U = spec.lstm_units
        cell = torch.nn.LSTMCell(X.shape[-1], U).double()
        del cell.weight_ih, cell.weight_hh, cell.bias_ih, cell.bias_hh
        cell.weight_ih, cell.weight_hh = P["lstm.wx"], P["lstm.wh"]
        cell.bias_ih, cell.bias_hh = P["lstm.b"], torch.zeros(4 * U, dtype=torch.float64)
        h = torch.tensor(batch["h0"], dtype=torch.float64)
        c = torch.tensor(batch["c0"], dtype=torch.float64)
        hs = []
        for t in range(T1):
            keep = (~done[:, t]).double()[:, None]
            h, c = cell(X[:, t], (h * keep, c * keep))
            hs.append(h)
        hfeat = torch.stack(hs, 1).reshape(B * T1, U)
    out = F.linear(hfeat, P["heads.w"], P["heads.b"])
    return out[:, :A].reshape(B, T1, A), out[:, A].reshape(B, T1), P


SPECS = {"c1": O.spec_c1, "c2": O.spec_c2, "c3": O.spec_c3, "c4": O.spec_c4}


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_network_fwd_bwd_vs_torch(cfg):
    spec = SPECS[cfg]()
    B, T = (3, 4) if cfg in ("c1", "c2") else (1, 2)
    batch = seedgen.learner_batch((16,) if cfg == "c1" else (spec.obs_h, spec.obs_w, spec.obs_c),
                                  spec.num_actions, B, T, seed=11,
                                  lstm_units=spec.lstm_units, done_p=0.3,
                                  float_obs=(cfg == "c1"), smm=(cfg == "c4"))
    flat = seedgen.glorot_params(O.param_layout(spec), seed=2, bias_std=0.1)
    P = O.unflatten(spec, flat)
    logits, values, cache = O.network_forward(spec, P, batch)
    tl, tv, TP = _torch_net(spec, flat, batch)
    np.testing.assert_allclose(logits, tl.detach().numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(values, tv.detach().numpy(), rtol=1e-10, atol=1e-12)
    g = seedgen.rng(3)
    dl = g.standard_normal(logits.shape)
    dv = g.standard_normal(values.shape)
    grads = O.network_backward(spec, P, batch, cache, dl, dv)
    ((tl * torch.tensor(dl)).sum() + (tv * torch.tensor(dv)).sum()).backward()
    for name, _ in O.param_layout(spec):
        ref = TP[name].grad.numpy()
        np.testing.assert_allclose(grads[name], ref, rtol=1e-9,
                                   atol=1e-11 * max(1.0, np.abs(ref).max()), err_msg=name)


def test_network_zero_params_S61_and_lstm_zero_S99():
    spec = O.spec_c2()
    batch = seedgen.learner_batch((84, 84, 4), 18, 2, 2, seed=1)
    batch["h0"][:] = 0
    batch["c0"][:] = 0
    P = O.unflatten(spec, np.zeros(O.param_count(spec)))
    logits, values, cache = O.network_forward(spec, P, batch)
    assert np.all(logits == 0) and np.all(values == 0)
    assert np.all(cache["lstm"]["c"] == 0)


def test_network_finite_difference_mlp_S72():
    spec = O.spec_c1()
    batch = seedgen.learner_batch((16,), 4, 2, 3, seed=4, lstm_units=0, float_obs=True)
    flat = seedgen.glorot_params(O.param_layout(spec), seed=1, bias_std=0.1).astype(np.float64)
    hp = dict(HP, loss_scale=1.0 / 6)

    def loss_at(f):
        P = O.unflatten(spec, f)
        lg, vl, _ = O.network_forward(spec, P, batch)
        return lg, vl

    lg, vl = loss_at(flat)
    L = O.policy_loss(lg, vl, batch["action"], batch["behaviour_logp"], batch["reward"],
                      batch["done"], hp)
    P = O.unflatten(spec, flat)
    _, _, cache = O.network_forward(spec, P, batch)
    grads = O.flatten(spec, O.network_backward(spec, P, batch, cache, L["dlogits"], L["dvalues"]))

    def frozen_loss(f):   # targets vs / pg_adv held constant
        lg2, vl2 = loss_at(f)
        T = lg2.shape[1] - 1
        logp = O.log_softmax(lg2[:, :T])
        a = batch["action"][:, :T].astype(np.int64)
        tl = np.take_along_axis(logp, a[:, :, None], 2)[:, :, 0]
        H = -(np.exp(logp) * logp).sum(-1)
        return hp["loss_scale"] * ((-L["pg_adv"] * tl).sum() + 0.25 * ((L["vs"] - vl2[:, :T]) ** 2).sum()
                                   - hp["ent_coef"] * H.sum())

    g = seedgen.rng(0)
    for i in g.choice(flat.size, 40, replace=False):
        e = np.zeros_like(flat)
        e[i] = 1e-6
        fd = (frozen_loss(flat + e) - frozen_loss(flat - e)) / 2e-6
        assert abs(fd - grads[i]) <= 1e-6 + 1e-5 * abs(fd), (i, fd, grads[i])


# ------------------------------------------------------------------ clip + Adam
def test_adam_and_clip_S81_S91():
    gold = _gold("nn_S81_S91.json")
    hp = dict(HP, lr=0.1, eps=1e-8, max_grad_norm=1e9)
    p, m, v, step, norm, applied = O.clip_adam(np.zeros(1), np.ones(1), np.zeros(1),
                                               np.zeros(1), 0, hp)
    assert p[0] == pytest.approx(gold["adam_w1"], rel=1e-6) and step == 1 and applied == 1
    # clip: the Adam step with lr->0 leaves params; check the clip scale via m (=(1-b1) g)
    hp = dict(HP, lr=0.0, max_grad_norm=1.0)
    _, m, _, _, norm, _ = O.clip_adam(np.zeros(2), np.array(gold["clip_in"]), np.zeros(2),
                                      np.zeros(2), 0, hp)
    assert norm == pytest.approx(5.0)
    np.testing.assert_allclose(m / (1 - hp["beta1"]), gold["clip_max1"], rtol=1e-12)
    hp = dict(HP, lr=0.0, max_grad_norm=10.0)
    _, m, _, _, _, _ = O.clip_adam(np.zeros(2), np.array(gold["clip_in"]), np.zeros(2),
                                   np.zeros(2), 0, hp)
    np.testing.assert_allclose(m / (1 - hp["beta1"]), gold["clip_in"], rtol=1e-12)


def test_adam_matches_torch_optim():
    g = seedgen.rng(8)
    p0 = g.standard_normal(50)
    hp = dict(HP, lr=1e-2, eps=1e-5, max_grad_norm=1e9)
    tp = torch.tensor(p0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tp], lr=hp["lr"], betas=(hp["beta1"], hp["beta2"]), eps=hp["eps"])
    p, m, v, step = p0.copy(), np.zeros(50), np.zeros(50), 0
    for k in range(3):
        gr = g.standard_normal(50)
        p, m, v, step, _, _ = O.clip_adam(p, gr, m, v, step, hp)
        tp.grad = torch.tensor(gr)
        opt.step()
    np.testing.assert_allclose(p, tp.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_nonfinite_grad_skips_update_S448():
    p, m, v, step, norm, applied = O.clip_adam(np.ones(3), np.array([1.0, np.nan, 0.0]),
                                               np.zeros(3), np.zeros(3), 4, HP)
    assert applied == 0 and step == 4 and np.all(p == 1.0)


# ------------------------------------------------------------------ DP semantics
def test_dp_gradient_is_sum_of_shards():
    """C20: an N-rank step (sum of per-shard grads, each scaled by 1/(N B T)) equals
    the single-process step on the concatenated batch."""
    spec = O.spec_c1()
    B, T, N = 2, 3, 2
    flat = seedgen.glorot_params(O.param_layout(spec), seed=3, bias_std=0.1)
    shards = [seedgen.learner_batch((16,), 4, B, T, seed=20 + i, lstm_units=0, float_obs=True)
              for i in range(N)]
    full = {k: np.concatenate([s[k] for s in shards], 0) for k in shards[0]}
    hp = dict(HP, loss_scale=1.0 / (N * B * T))
    z = np.zeros(flat.size)
    whole = O.learner_step(spec, flat, z, z, 0, full, hp)
    parts = [O.learner_step(spec, flat, z, z, 0, s, hp)["grads"] for s in shards]
    np.testing.assert_allclose(whole["grads"], parts[0] + parts[1], rtol=1e-12, atol=1e-15)


# ------------------------------------------------------------------ inference
def test_inverse_cdf_sampling_C18():
    logits = np.log(np.array([[0.1, 0.2, 0.3, 0.4]] * 5))
    u = np.array([0.05, 0.15, 0.35, 0.65, 0.9999])
    np.testing.assert_array_equal(O.sample_inverse_cdf(logits, u), [0, 1, 2, 3, 3])


def test_infer_state_semantics_S440_S441():
    spec = O.spec_c2()
    flat = seedgen.glorot_params(O.param_layout(spec), seed=5, bias_std=0.1)
    NA, U = 16, 256
    g = seedgen.rng(2)
    th = g.standard_normal((NA, U))
    tc = g.standard_normal((NA, U))
    tla = g.integers(0, 18, NA)
    req = seedgen.infer_requests((84, 84, 4), 18, NA, 4, seed=1)
    req["done"][:] = [1, 0, 1, 0]
    a, blp, lg, th2, tc2, tla2 = O.infer(spec, flat, th, tc, tla, req["actor_ids"], req["obs"],
                                         req["reward"], req["done"], req["uniforms"])
    others = np.setdiff1d(np.arange(NA), req["actor_ids"])
    np.testing.assert_array_equal(th2[others], th[others])      # untouched (bitwise)
    np.testing.assert_array_equal(tla2[req["actor_ids"]], a)
    # done=1 -> identical to a fresh actor with zero state and no previous action
    th0, tc0 = th.copy(), tc.copy()
    th0[req["actor_ids"][0]] = 0
    tc0[req["actor_ids"][0]] = 0
    tla0 = tla.copy()
    tla0[req["actor_ids"][0]] = -1
    req2 = {k: v[:1].copy() for k, v in req.items()}
    req2["done"][:] = 0
    req2["reward"][:] = 0
    a2, blp2, lg2, _, _, _ = O.infer(spec, flat, th0, tc0, tla0, req2["actor_ids"], req2["obs"],
                                     req2["reward"], req2["done"], req2["uniforms"])
    np.testing.assert_allclose(lg2[0], lg[0], rtol=1e-12)
    assert np.isclose(blp[0], np.log(np.exp(O.log_softmax(lg[:1]))[0, a[0]]))


def test_unroll_accounting_S442():
    """unroll length 4: the 5th step completes a trajectory (steps 1-4 + step 5 as
    bootstrap), and the next unroll restarts containing step 5."""
    st = O.UnrollStore(T=4, num_actors=1)
    for k in range(5):
        st.record(0, {"step": k + 1}, np.zeros(1) + k, np.zeros(1))
    assert st.ready == [(0, 0)]
    assert [s["step"] for s in st.steps[(0, 0)]["slots"]] == [1, 2, 3, 4, 5]
    assert [s["step"] for s in st.steps[(0, 1)]["slots"]] == [5]
    assert st.steps[(0, 1)]["h0"][0] == 4        # state before step 5 (C19)


# ------------------------------------------------------------------ bf16 emulation (C26)
def test_bf16_round_matches_torch_bfloat16():
    g = seedgen.rng(12)
    x = np.concatenate([g.standard_normal(10000) * 10.0 ** g.integers(-30, 30, 10000),
                        [0.0, -0.0, 1.0, 1.00390625, 1.01171875, 65504.0, 3.0e38]])
    ref = torch.tensor(x.astype(np.float32)).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(O.bf16_round(x), ref)


def test_emulated_oracle_stays_close_to_exact():
    """The bf16-emulated forward differs from the exact fp64 definition only by
    bf16 rounding (a few 1e-3 relative on the outputs)."""
    spec = O.spec_c2()
    batch = seedgen.learner_batch((84, 84, 4), 18, 2, 3, seed=3, done_p=0.2)
    P = O.unflatten(spec, seedgen.glorot_params(O.param_layout(spec), seed=4, bias_std=0.1))
    le, ve, _ = O.network_forward(spec, P, batch, emu=True)
    lx, vx, _ = O.network_forward(spec, P, batch, emu=False)
    assert np.linalg.norm(le - lx) / np.linalg.norm(lx) < 2e-2
    assert np.linalg.norm(ve - vx) / np.linalg.norm(vx) < 2e-2


def test_philox4x32_10_known_answers():
    g = _gold("philox4x32_10_kat.json")
    for v in g["vectors"]:
        out = O.philox4x32_10([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert [int(x) for x in out] == [int(x, 16) for x in v["out"]]
    u = O.philox_uniforms(7, 3, np.arange(1000))
    assert np.all((u >= 0) & (u < 1)) and abs(u.mean() - 0.5) < 0.05


# ------------------------------------------------------------------ R2D2
def test_value_rescale_golden_S206_and_roundtrip():
    """S:206-207 printed values rescale(3) = 1.003, rescale(-3) = -1.003, rescale(0) = 0;
    S:238 invariant h^-1(h(x)) = x over |x| <= 1e4 (the two functions checked
    against each other, h increasing and odd)."""
    assert O.value_rescale(0.0) == 0.0
    assert abs(O.value_rescale(3.0) - 1.003) < 1e-12
    assert abs(O.value_rescale(-3.0) + 1.003) < 1e-12
    x = np.concatenate([np.linspace(-1e4, 1e4, 20001), seedgen.rng(5).normal(0, 30, 1000)])
    assert np.max(np.abs(O.value_rescale_inv(O.value_rescale(x)) - x)) < 1e-5
    h = O.value_rescale(np.sort(x))
    assert np.all(np.diff(h) >= 0) and np.allclose(O.value_rescale(-x), -O.value_rescale(x))


def _r2d2_case(B, T, A, seed, done_p=0.1):
    g = seedgen.rng(seed)
    qo = g.normal(0, 1.5, (B, T + 1, A))
    qt = g.normal(0, 1.5, (B, T + 1, A))
    a = g.integers(0, A, (B, T + 1))
    r = g.normal(0, 1, (B, T)) * (g.random((B, T)) < 0.3)
    disc = 0.997 * (g.random((B, T)) >= done_p)
    return qo, qt, a, r, disc


def test_r2d2_targets_terminal_and_priority_goldens_S218_S227():
    """terminal step (discount 0) with r = 1 -> y = rescale(1) = 0.41521;
    S:227: |delta| = [1, 3], eta = 0.9 -> priority 2.9."""
    qo = np.zeros((1, 2, 3))
    qt = np.full((1, 2, 3), 7.0)                 # never used: the bootstrap is discounted away
    y, d, p = O.r2d2_targets(qo, qt, np.zeros((1, 2), int), np.array([[1.0]]),
                             np.array([[0.0]]), n=5)
    assert abs(y[0, 0] - 0.41521356237309515) < 1e-12
    # two steps, both terminal, rewards r: y_t = h(r_t); q chosen so delta = [1, -3]
    r = np.array([[2.0, -5.0]])
    qo = np.zeros((1, 3, 2))
    qo[0, 0, 0] = O.value_rescale(2.0) - 1.0
    qo[0, 1, 1] = O.value_rescale(-5.0) + 3.0
    y, d, p = O.r2d2_targets(qo, qo, np.array([[0, 1, 0]]), r, np.zeros((1, 2)), n=5, eta=0.9)
    np.testing.assert_allclose(d, [[1.0, -3.0]], atol=1e-12)
    assert abs(p[0] - 2.9) < 1e-12


def test_r2d2_targets_geometric_closed_form():
    """Constant reward r, constant gamma, no episode end, all Q = 0: the n-step return
    is the geometric sum r (1 - gamma^m) / (1 - gamma), m = min(n, T - t), and h^-1(0) = 0."""
    B, T, A, n, gam, rv = 2, 9, 4, 5, 0.97, 0.7
    z = np.zeros((B, T + 1, A))
    y, _, _ = O.r2d2_targets(z, z, np.zeros((B, T + 1), int), np.full((B, T), rv),
                             np.full((B, T), gam), n=n)
    for t in range(T):
        m = min(n, T - t)
        np.testing.assert_allclose(y[:, t], O.value_rescale(rv * (1 - gam ** m) / (1 - gam)),
                                   rtol=1e-12)


def test_r2d2_double_q_decoupling_S241():
    """Perturbing q_target at actions other than the online argmax leaves y unchanged;
    perturbing it at the argmax changes y (double Q: online selects, target evaluates)."""
    qo, qt, a, r, disc = _r2d2_case(3, 12, 6, seed=3)
    y0, _, _ = O.r2d2_targets(qo, qt, a, r, disc, n=5)
    amax = qo.argmax(-1)
    mask = np.ones_like(qt, bool)
    np.put_along_axis(mask, amax[..., None], False, axis=2)
    y1, _, _ = O.r2d2_targets(qo, np.where(mask, qt + 9.0, qt), a, r, disc, n=5)
    np.testing.assert_array_equal(y0, y1)
    y2, _, _ = O.r2d2_targets(qo, np.where(mask, qt, qt + 1.0), a, r, disc, n=5)
    assert np.mean(np.abs(y2 - y0) > 0) > 0.5     # (zero only where an episode end drops it)


def test_r2d2_nstep_recursion_equals_window_sum():
    """The n-step return as the recursion G^(k)_t = r_t + gamma_t G^(k-1)_{t+1},
    G^(0)_s = h^-1(q_target[s][argmax q_online[s]]) (written here independently of
    the oracle's forward window sum) gives the same y."""
    qo, qt, a, r, disc = _r2d2_case(2, 11, 5, seed=4)
    n = 4
    y, _, _ = O.r2d2_targets(qo, qt, a, r, disc, n=n)
    B, T = r.shape
    boot = O.value_rescale_inv(np.take_along_axis(qt, qo.argmax(-1)[..., None], 2)[..., 0])

    def G(b, t, k):
        return boot[b, t] if k == 0 else r[b, t] + disc[b, t] * G(b, t + 1, k - 1)
    for b in range(B):
        for t in range(T):
            assert abs(O.value_rescale(G(b, t, min(n, T - t))) - y[b, t]) < 1e-12


def test_r2d2_loss_grad_vs_autograd():
    qo, qt, a, r, disc = _r2d2_case(2, 6, 4, seed=6)
    y, _, _ = O.r2d2_targets(qo, qt, a, r, disc, n=3)
    w = np.array([0.7, 1.0])
    loss, dq = O.r2d2_loss_grad(qo, a, y, w, 0.25)
    q = torch.tensor(qo, requires_grad=True)
    taken = torch.gather(q[:, :-1], 2, torch.tensor(a[:, :-1])[..., None])[..., 0]
    L = 0.25 * (torch.tensor(w)[:, None] * 0.5 * (taken - torch.tensor(y)) ** 2).sum()
    L.backward()
    assert abs(L.item() - loss) < 1e-12
    np.testing.assert_allclose(dq, q.grad.numpy(), atol=1e-14)


def test_replay_probabilities_golden_S313_and_sampling():
    """priorities [1, 16], alpha = 0.9 -> P ~ [0.0762, 0.9238]; equal priorities ->
    all weights 1; a zero priority is never drawn; 100k inverse-CDF draws pass a
    chi-square goodness-of-fit against p^alpha / sum (significance 0.001)."""
    P = O.replay_probabilities([1.0, 16.0], 0.9)
    np.testing.assert_allclose(P, [0.0762, 0.9238], atol=5e-5)
    idx, w = O.replay_sample([2.0] * 5, np.linspace(0, 0.999, 50), 0.9, 0.6)
    np.testing.assert_allclose(w, 1.0)
    assert set(idx) == set(range(5))
    idx, _ = O.replay_sample([0.0, 1.0], seedgen.rng(1).random(1000))
    assert np.all(idx == 1)
    from scipy.stats import chisquare
    pr = seedgen.rng(2).random(40) * 5
    idx, _ = O.replay_sample(pr, seedgen.rng(3).random(100000), 0.9, 0.6)
    obs = np.bincount(idx, minlength=40)
    exp = O.replay_probabilities(pr, 0.9) * 100000
    assert chisquare(obs, exp).pvalue > 1e-3


def test_r2d2_learner_step_finite_differences():
    """The R2D2 learner-step oracle's gradient = central differences of its loss with
    the targets y and the burn-in states held constant (stop-gradient targets;
    burn-in without gradient), on the Atari net (fp64, h = 1e-6), at sampled
    coordinates of every layer type — pins the dueling backward and the gradient
    cut at the burn-in boundary."""
    spec = O.spec_c2(num_actions=5)
    layout = O.param_layout(spec)
    params = seedgen.glorot_params(layout, seed=3, bias_std=0.1).astype(np.float64)
    tparams = seedgen.glorot_params(layout, seed=4, bias_std=0.1).astype(np.float64)
    B, bi, T = 2, 3, 4
    full = seedgen.learner_batch((84, 84, 4), 5, B, bi + T, seed=5, done_p=0.1)
    burn = {k: (v[:, :bi] if v.ndim >= 2 and v.shape[1] == bi + T + 1 else v) for k, v in full.items()}
    train = {k: (v[:, bi:] if v.ndim >= 2 and v.shape[1] == bi + T + 1 else v) for k, v in full.items()}
    hp = dict(discount=0.997, n=3, eta=0.9, rescale_eps=1e-3, loss_scale=1.0 / (B * T), lr=1e-4,
              beta1=0.9, beta2=0.999, eps=1e-3, max_grad_norm=80.0)
    w = np.array([0.6, 1.0])
    z = np.zeros(params.size)
    ref = O.r2d2_learner_step(spec, params, tparams, z, z, 0, burn, train, w, hp)
    h0, c0 = ref["warm"]
    y = ref["y"]
    tr = dict(train, h0=h0, c0=c0)

    def loss(pv):
        lo, vo, _ = O.network_forward(spec, O.unflatten(spec, pv), tr)
        return O.r2d2_loss_grad(O.dueling_q(lo, vo), train["action"], y, w, hp["loss_scale"])[0]
    offs = {n: o for (n, _), o in zip(layout, np.cumsum([0] + [int(np.prod(s)) for _, s in layout])[:-1])}
    g = seedgen.rng(6)
    for name in ("heads.w", "heads.b", "lstm.wh", "lstm.wx", "lstm.b", "fc.w", "conv2.w", "conv1.b"):
        size = int(np.prod(dict(layout)[name]))
        for k in g.choice(size, 2, replace=False):
            i = offs[name] + k
            e = np.zeros(params.size)
            e[i] = 1e-6
            fd = (loss(params + e) - loss(params - e)) / 2e-6
            assert abs(fd - ref["grads"][i]) <= 1e-6 + 1e-4 * abs(fd), (name, k, fd, ref["grads"][i])


def test_actor_epsilon_P614_and_eps_greedy():
    """epsilon_i = 0.4^(1 + 7 i / (N - 1)) — the first actor explores at 0.4, the
    last at 0.4^8; epsilon-greedy: the behaviour probabilities of one state sum to 1
    over the actions (enumerated through the uniform draws), the greedy action gets
    1 - eps + eps/A, ties go to the first maximum."""
    assert O.actor_epsilon(0, 610) == pytest.approx(0.4, abs=0)
    assert O.actor_epsilon(609, 610) == pytest.approx(0.4 ** 8, rel=1e-15)
    assert O.actor_epsilon(0, 1) == 0.4
    assert O.actor_epsilon(3, 7) == pytest.approx(0.4 ** (1 + 7 * 3 / 6), rel=1e-15)
    q = np.array([0.5, 2.0, -1.0, 2.0])
    eps = 0.3
    # greedy branch: first maximum
    a, p = O.eps_greedy_action(q, eps, u_explore=0.9, u_action=0.0)
    assert a == 1 and p == pytest.approx(eps / 4 + 1 - eps)
    # explore branch: floor(u * A), clamped
    assert O.eps_greedy_action(q, eps, 0.1, 0.0)[0] == 0
    assert O.eps_greedy_action(q, eps, 0.1, 0.74)[0] == 2
    assert O.eps_greedy_action(q, eps, 0.1, 1.0)[0] == 3
    # the behaviour distribution, enumerated over a fine grid of (u0, u1), sums to 1 and
    # matches the returned probabilities
    g = (np.arange(200) + 0.5) / 200
    freq = np.zeros(4)
    for u0 in g:
        for u1 in g:
            freq[O.eps_greedy_action(q, eps, u0, u1)[0]] += 1
    freq /= freq.sum()
    probs = np.array([eps / 4 + (1 - eps) * (k == 1) for k in range(4)])
    np.testing.assert_allclose(freq, probs, atol=1e-12)
    assert probs.sum() == pytest.approx(1.0)
