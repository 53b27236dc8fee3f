"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no softmax, no V-trace, no
network math): it only draws seeded random tensors with the shapes, value
distributions and structure of the paper's workloads (recipe: DESIGN.md §5,
SURVEY.md §8(d)).  Both sides receive the same bytes from here.
"""
from __future__ import annotations

import numpy as np

ATARI_OBS = (84, 84, 4)        # P:624-648 (only the shape is used)
DMLAB_OBS = (72, 96, 3)        # BJ configs[2]
SMM_OBS = (72, 96, 16)         # P:358 + BJ configs[3] (4 planes x 4 stacked frames)


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def vtrace_inputs(B, T, seed=0, done_p=1.0 / 200, gamma=0.99, value_scale=3.0,
                  force_done_at=None):
    """V-trace call inputs, all float32 [B][T] (+ bootstrap [B]).

    behaviour log-prob  = -log(A) + N(0, 0.5^2) (clipped to <= 0), A = 18
    target log-prob     = behaviour + N(0, 0.3^2)  ("near on-policy")
    rewards             = N(0,1) * Bernoulli(0.1)  (sparse)
    discounts           = gamma * (1 - done), done ~ Bernoulli(done_p)
    values, bootstrap   ~ N(0, value_scale^2)
    """
    g = rng(seed)
    blp = np.minimum(-np.log(18.0) + 0.5 * g.standard_normal((B, T)), 0.0)
    tlp = np.minimum(blp + 0.3 * g.standard_normal((B, T)), 0.0)
    r = g.standard_normal((B, T)) * (g.random((B, T)) < 0.1)
    done = g.random((B, T)) < done_p
    if force_done_at is not None:
        done[:, force_done_at] = True
    disc = gamma * (1.0 - done)
    V = value_scale * g.standard_normal((B, T))
    boot = value_scale * g.standard_normal(B)
    f = lambda x: np.ascontiguousarray(x, dtype=np.float32)
    return dict(behaviour_logp=f(blp), target_logp=f(tlp), rewards=f(r), discounts=f(disc),
                values=f(V), bootstrap=f(boot))


def glorot_params(layout, seed=0, bias_std=0.0, forget_bias=1.0, lstm_units=256):
    """Flat float32 params for an ordered layout [(name, shape)].

    Weights: Glorot uniform, limit sqrt(6/(fan_in+fan_out)) with
    fan_in = prod(shape[1:]), fan_out = shape[0] * prod(shape[1:-1]) for
    conv kernels [O][KH][KW][C] and shape[0] for dense [O][I].
    Biases: N(0, bias_std^2) (0 = zeros); the LSTM forget-gate slice gets
    +forget_bias (C14 init recipe).
    """
    g = rng(seed)
    out = []
    for name, shape in layout:
        shape = tuple(shape)
        if len(shape) == 1:
            b = bias_std * g.standard_normal(shape) if bias_std else np.zeros(shape)
            if name == "lstm.b":
                b[lstm_units:2 * lstm_units] += forget_bias
            out.append(b)
            continue
        rf = int(np.prod(shape[1:-1])) if len(shape) > 2 else 1
        fan_in = int(np.prod(shape[1:]))
        fan_out = shape[0] * rf
        lim = np.sqrt(6.0 / (fan_in + fan_out))
        out.append(g.uniform(-lim, lim, size=shape))
    return np.ascontiguousarray(np.concatenate([o.ravel() for o in out]), dtype=np.float32)


def learner_batch(obs_shape, num_actions, B, T, seed=0, lstm_units=256, done_p=1.0 / 200,
                  smm=False, float_obs=False, force_done=()):
    """One [B][T+1] unroll batch in the seed_batch layout (include/seed.h).

    obs: uint8 uniform 0..255 (Atari / DMLab); SMM planes binary {0,255} with
    ~2% ones (smm=True); float32 N(0,1) for the MLP config (float_obs=True).
    action ~ U{0..A-1}; prev_action[t] = action[t-1], prev_action[0] ~ U{-1..A-1};
    reward = N(0,1) * Bernoulli(0.1); done ~ Bernoulli(done_p) (+ forced (b,t));
    behaviour_logp = -log(A) + N(0, 0.3^2); h0, c0 ~ N(0, 0.1^2).
    """
    g = rng(seed)
    T1 = T + 1
    if float_obs:
        obs = g.standard_normal((B, T1) + tuple(obs_shape)).astype(np.float32)
    elif smm:
        obs = ((g.random((B, T1) + tuple(obs_shape)) < 0.02) * 255).astype(np.uint8)
    else:
        obs = g.integers(0, 256, size=(B, T1) + tuple(obs_shape), dtype=np.uint8)
    action = g.integers(0, num_actions, size=(B, T1)).astype(np.int32)
    prev = np.empty_like(action)
    prev[:, 1:] = action[:, :-1]
    prev[:, 0] = g.integers(-1, num_actions, size=B)
    reward = (g.standard_normal((B, T1)) * (g.random((B, T1)) < 0.1)).astype(np.float32)
    done = (g.random((B, T1)) < done_p)
    for (b, t) in force_done:
        done[b, t] = True
    blp = (-np.log(num_actions) + 0.3 * g.standard_normal((B, T1))).astype(np.float32)
    U = max(lstm_units, 1)
    h0 = (0.1 * g.standard_normal((B, U))).astype(np.float32)
    c0 = (0.1 * g.standard_normal((B, U))).astype(np.float32)
    return dict(obs=np.ascontiguousarray(obs), action=action, prev_action=prev, reward=reward,
                done=done.astype(np.uint8), behaviour_logp=blp, h0=h0, c0=c0)


def infer_requests(obs_shape, num_actions, num_actors, n, seed=0, call_index=0,
                   done_p=1.0 / 200):
    """One inference call: n unique actor ids (next slice of a seeded permutation),
    uint8 obs, rewards N(0,1)*Bern(0.1), done ~ Bern(done_p), uniforms U[0,1)."""
    g = rng(seed * 1000003 + call_index)
    perm = rng(seed).permutation(num_actors)
    start = (call_index * n) % num_actors
    ids = np.resize(np.roll(perm, -start), n).astype(np.int32)
    obs = g.integers(0, 256, size=(n,) + tuple(obs_shape), dtype=np.uint8)
    reward = (g.standard_normal(n) * (g.random(n) < 0.1)).astype(np.float32)
    done = (g.random(n) < done_p).astype(np.uint8)
    u = g.random(n).astype(np.float32)
    return dict(actor_ids=ids, obs=obs, reward=reward, done=done, uniforms=u)
