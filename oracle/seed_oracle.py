"""SEED learner / inference oracle — plain, slow, obviously-correct fp64 numpy.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_1910_06591_b200``) never imports it and
shares no code with it: the two sides meet only through the seeded input
generators in ``seedgen/`` (which hold none of the method's arithmetic) and
through the flat layouts documented in ``include/seed.h``.

Citations: ``P:NNN`` = line of /root/reference/PAPER.md, ``S:NNN`` = line of
/root/reference/SPEC.md, ``C#`` = reading # of SURVEY.md §8(c) / DESIGN.md §3.
Every function computes in float64 from the given (fp32 / uint8) input bytes.

What each function follows
--------------------------
* ``vtrace``          S:140 recursion (the IMPALA V-trace definition cited at
                      P:143-145; PAPER.md prints no formula, reading C1).
* ``vtrace_direct``   the O(T^2) sum form of the same definition (C1).
* ``policy_loss``     S:149-157 loss decomposition, H7 closed-form gradients.
* network fwd/bwd     direct-definition conv / max-pool / dense / LSTM
                      (P:591 core inputs, S:47/S:57 reset, C14/C15 layer lists).
* ``clip_adam``       S:75-93 (textbook Adam with bias correction, global-norm clip).
* ``infer``           S:434-442 serve_inference semantics (C17-C19 readings).

Parity status of each function is listed in DESIGN.md §4; every function here is
pinned by a ``-m "not gpu"`` test in tests/test_oracle_pins.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------
# bf16 emulation (reading C26): the tensor-core path rounds GEMM operands and
# stored activations / gradients to bf16 (round-to-nearest-even).  A ReLU mask
# is a floating-point decision of an integer (a mask bit), so parity compares
# the kernels with this oracle taking the same decisions at the same rounding
# points ("emu" mode); "exact" mode is the plain fp64 definition.
# --------------------------------------------------------------------------
def bf16_round(x):
    """Round to the nearest bf16 (ties to even), via the float32 bit pattern."""
    f = np.ascontiguousarray(np.asarray(x, np.float64).astype(np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(x))


def _q(x, emu):
    return bf16_round(x) if emu else x


# --------------------------------------------------------------------------
# network specs (C14) — the architecture definitions, independent of the GPU
# side's own definitions in include/seed.h.
# --------------------------------------------------------------------------
NET_MLP, NET_ATARI_SHALLOW, NET_IMPALA_DEEP, NET_GFOOTBALL = 0, 1, 2, 3


@dataclass
class NetSpec:
    kind: int
    obs_h: int
    obs_w: int
    obs_c: int
    num_actions: int
    lstm_units: int = 256
    mlp_hidden: tuple = (64, 64)
    sections: tuple = ()          # IMPALA-deep channel list (C14)

    @property
    def obs_dim(self):
        return self.obs_h * self.obs_w * self.obs_c


def spec_c1():
    """BJ configs[0]: tiny 2-layer MLP, 16-d obs, 4 actions, fp32, feed-forward."""
    return NetSpec(NET_MLP, 1, 1, 16, 4, lstm_units=0)


def spec_c2(num_actions=18):
    """BJ configs[1]: Atari IMPALA-shallow CNN (C14) + LSTM256, 84x84x4 uint8."""
    return NetSpec(NET_ATARI_SHALLOW, 84, 84, 4, num_actions)


def spec_c3(num_actions=15, width=1):
    """BJ configs[2]: DMLab IMPALA deep ResNet (16,32,32) + LSTM256, 72x96x3; width 2 =
    the "Medium 2x" filters (32, 64, 64) of P:411."""
    return NetSpec(NET_IMPALA_DEEP, 72, 96, 3, num_actions,
                   sections=tuple(width * c for c in (16, 32, 32)))


def spec_c3_medium(num_actions=15):
    """P:411 DMLab Medium: 2x filters."""
    return spec_c3(num_actions, width=2)


def spec_c3_large(num_actions=15):
    """P:411, P:434 DMLab Large: 4x filters (64, 128, 128)."""
    return spec_c3(num_actions, width=4)


def spec_c4(num_actions=19, obs_h=72, obs_w=96):
    """BJ configs[3]: GRF SMM 72x96x16, IMPALA-deep block (16,32,32,32) + LSTM256.
    P:358: the SMM is 96 x 72 by default, Medium 120 x 90, Large 144 x 108
    (width x height)."""
    return NetSpec(NET_GFOOTBALL, obs_h, obs_w, 16, num_actions, sections=(16, 32, 32, 32))


def spec_c4_medium(num_actions=19):
    """P:358 Medium SMM: 120 x 90 (W x H)."""
    return spec_c4(num_actions, obs_h=90, obs_w=120)


def spec_c4_large(num_actions=19):
    """P:358 Large SMM: 144 x 108 (W x H)."""
    return spec_c4(num_actions, obs_h=108, obs_w=144)


def _same_out(n, s):
    return -(-n // s)


def torso_out_shape(spec):
    """(H, W, C) of the torso output before the FC layer."""
    if spec.kind == NET_ATARI_SHALLOW:
        h1 = (spec.obs_h - 8) // 4 + 1
        w1 = (spec.obs_w - 8) // 4 + 1
        h2 = (h1 - 4) // 2 + 1
        w2 = (w1 - 4) // 2 + 1
        return h2, w2, 32
    if spec.kind in (NET_IMPALA_DEEP, NET_GFOOTBALL):
        h, w = spec.obs_h, spec.obs_w
        for _ in spec.sections:
            h, w = _same_out(h, 2), _same_out(w, 2)
        return h, w, spec.sections[-1]
    raise ValueError(spec.kind)


def param_layout(spec):
    """Ordered list of (name, shape).  Flat fp32 params are these tensors,
    row-major, concatenated in this order (the order include/seed.h documents)."""
    A = spec.num_actions
    out = []
    if spec.kind == NET_MLP:
        d = spec.obs_dim
        for i, hdim in enumerate(spec.mlp_hidden):
            out += [(f"mlp{i}.w", (hdim, d)), (f"mlp{i}.b", (hdim,))]
            d = hdim
        out += [("heads.w", (A + 1, d)), ("heads.b", (A + 1,))]
        return out
    if spec.kind == NET_ATARI_SHALLOW:
        out += [("conv1.w", (16, 8, 8, spec.obs_c)), ("conv1.b", (16,)),
                ("conv2.w", (32, 4, 4, 16)), ("conv2.b", (32,))]
    else:
        cin = spec.obs_c
        for s, ch in enumerate(spec.sections):
            out += [(f"s{s}.conv.w", (ch, 3, 3, cin)), (f"s{s}.conv.b", (ch,))]
            for r in range(2):
                for j in range(2):
                    out += [(f"s{s}.res{r}.conv{j}.w", (ch, 3, 3, ch)),
                            (f"s{s}.res{r}.conv{j}.b", (ch,))]
            cin = ch
    h, w, c = torso_out_shape(spec)
    out += [("fc.w", (256, h * w * c)), ("fc.b", (256,))]
    U = spec.lstm_units
    core_in = 256 + A + 1
    out += [("lstm.wx", (4 * U, core_in)), ("lstm.wh", (4 * U, U)), ("lstm.b", (4 * U,))]
    out += [("heads.w", (A + 1, U)), ("heads.b", (A + 1,))]
    return out


def param_count(spec):
    return sum(int(np.prod(s)) for _, s in param_layout(spec))


def unflatten(spec, flat):
    flat = np.asarray(flat, dtype=np.float64)
    out, off = {}, 0
    for name, shape in param_layout(spec):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    assert off == flat.size, (off, flat.size)
    return out


def flatten(spec, tensors):
    return np.concatenate([np.asarray(tensors[name], dtype=np.float64).ravel()
                           for name, _ in param_layout(spec)])


# --------------------------------------------------------------------------
# V-trace (H6).  S:140; IMPALA definition cited at P:143-145 (reading C1-C7).
# --------------------------------------------------------------------------
def vtrace(behaviour_logp, target_logp, rewards, discounts, values, bootstrap,
           rho_bar=1.0, c_bar=1.0, lam=1.0):
    """Backward recursion of S:140, arrays [B][T], bootstrap [B].

    ratio_t = exp(tlp_t - blp_t); rho_t = min(rho_bar, ratio_t);
    c_t = lam * min(c_bar, ratio_t); delta_t = rho_t (r_t + g_t V_{t+1} - V_t)
    with V_T := bootstrap; v_t - V_t = delta_t + g_t c_t (v_{t+1} - V_{t+1}),
    v_T - V_T := 0 (C4); pg_adv_t = rho_t (r_t + g_t v_{t+1} - V_t), v_T := bootstrap.
    Returns (vs, pg_adv, nonfinite) — nonfinite per S:143 / C7.
    """
    blp = np.asarray(behaviour_logp, np.float64)
    tlp = np.asarray(target_logp, np.float64)
    r = np.asarray(rewards, np.float64)
    g = np.asarray(discounts, np.float64)
    V = np.asarray(values, np.float64)
    boot = np.asarray(bootstrap, np.float64)
    B, T = V.shape
    with np.errstate(over="ignore", invalid="ignore"):
        diff = tlp - blp
        ratio = np.exp(diff)
        rho = np.minimum(rho_bar, ratio)
        c = lam * np.minimum(c_bar, ratio)
        V_next = np.concatenate([V[:, 1:], boot[:, None]], axis=1)
        delta = rho * (r + g * V_next - V)
        vs = np.empty_like(V)
        acc = np.zeros(B)
        for t in range(T - 1, -1, -1):
            acc = delta[:, t] + g[:, t] * c[:, t] * acc
            vs[:, t] = V[:, t] + acc
        vs_next = np.concatenate([vs[:, 1:], boot[:, None]], axis=1)
        pg_adv = rho * (r + g * vs_next - V)
    nonfinite = not (np.all(np.isfinite(diff)) and np.all(np.isfinite(r)) and
                     np.all(np.isfinite(g)) and np.all(np.isfinite(V)) and
                     np.all(np.isfinite(boot)))
    return vs, pg_adv, nonfinite


def vtrace_direct(behaviour_logp, target_logp, rewards, discounts, values, bootstrap,
                  rho_bar=1.0, c_bar=1.0, lam=1.0):
    """The O(T^2) sum form (IMPALA eq. 1, reading C1):
    v_s = V_s + sum_{t>=s} (prod_{i=s}^{t-1} g_i c_i) delta_t."""
    blp = np.asarray(behaviour_logp, np.float64)
    tlp = np.asarray(target_logp, np.float64)
    r = np.asarray(rewards, np.float64)
    g = np.asarray(discounts, np.float64)
    V = np.asarray(values, np.float64)
    boot = np.asarray(bootstrap, np.float64)
    B, T = V.shape
    ratio = np.exp(tlp - blp)
    rho = np.minimum(rho_bar, ratio)
    c = lam * np.minimum(c_bar, ratio)
    Vn = np.concatenate([V[:, 1:], boot[:, None]], axis=1)
    delta = rho * (r + g * Vn - V)
    vs = np.empty_like(V)
    for s in range(T):
        total = np.zeros(B)
        for t in range(s, T):
            coef = np.ones(B)
            for i in range(s, t):
                coef = coef * g[:, i] * c[:, i]
            total = total + coef * delta[:, t]
        vs[:, s] = V[:, s] + total
    vsn = np.concatenate([vs[:, 1:], boot[:, None]], axis=1)
    return vs, rho * (r + g * vsn - V)


# --------------------------------------------------------------------------
# Loss and output gradients (H5, H7).  S:149-157; P:550 (c_v), P:545 (c_e).
# --------------------------------------------------------------------------
def log_softmax(z):
    m = z.max(axis=-1, keepdims=True)
    return z - m - np.log(np.exp(z - m).sum(axis=-1, keepdims=True))


def policy_loss(logits, values, actions, behaviour_logp, rewards, dones, hp):
    """Loss over one [B][T+1] unroll batch (layout of seed_batch, reading C5).

    logits [B][T+1][A], values [B][T+1] (network outputs); actions, rewards,
    dones, behaviour_logp [B][T+1] (batch tensors).  Trained steps t = 0..T-1:
      log pi(a_t|x_t), H_t from logits[:, t]; reward for a_t = rewards[:, t+1];
      discount g_t = gamma * (1 - dones[:, t+1]); V_t = values[:, t];
      bootstrap = values[:, T]  (C5).
    L = s * sum_{b,t<T} [ -pg_adv log pi(a_t) + 1/2 c_v (vs_t - V_t)^2 - c_e H_t ]  (C8-C10)
    Returns dict with loss parts, vs, pg_adv, dlogits [B][T+1][A], dvalues [B][T+1].
    """
    z = np.asarray(logits, np.float64)
    V = np.asarray(values, np.float64)
    B, T1, A = z.shape
    T = T1 - 1
    act = np.asarray(actions)[:, :T].astype(np.int64)
    logp = log_softmax(z[:, :T])
    p = np.exp(logp)
    tlp = np.take_along_axis(logp, act[:, :, None], axis=2)[:, :, 0]
    H = -(p * logp).sum(axis=-1)
    disc = hp["discount"] * (1.0 - np.asarray(dones, np.float64)[:, 1:])
    r = np.asarray(rewards, np.float64)[:, 1:]
    vs, pg_adv, nonfinite = vtrace(np.asarray(behaviour_logp, np.float64)[:, :T], tlp, r,
                                   disc, V[:, :T], V[:, T], hp["rho_bar"], hp["c_bar"],
                                   hp["lambda"])
    s = hp["loss_scale"]
    cv, ce = hp["vf_coef"], hp["ent_coef"]
    pg_loss = s * np.sum(-pg_adv * tlp)
    base_loss = s * 0.5 * cv * np.sum((vs - V[:, :T]) ** 2)
    ent_loss = -s * ce * np.sum(H)
    onehot = np.zeros_like(p)
    np.put_along_axis(onehot, act[:, :, None], 1.0, axis=2)
    dlogits = np.zeros_like(z)
    dlogits[:, :T] = s * (-pg_adv[:, :, None] * (onehot - p) + ce * p * (logp + H[:, :, None]))
    dvalues = np.zeros_like(V)
    dvalues[:, :T] = s * cv * (V[:, :T] - vs)
    return dict(loss=pg_loss + base_loss + ent_loss, pg=pg_loss, baseline=base_loss,
                entropy=ent_loss, vs=vs, pg_adv=pg_adv, target_logp=tlp, entropy_t=H,
                dlogits=dlogits, dvalues=dvalues, nonfinite=nonfinite)


# --------------------------------------------------------------------------
# Layer definitions (direct sums) and their hand-derived backward passes.
# Images are NHWC float64; conv weights [Cout][KH][KW][Cin] (C14).
# --------------------------------------------------------------------------
def relu(x):
    return np.maximum(x, 0.0)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def conv2d(x, w, b, stride, pad):
    """y[n,oy,ox,o] = b[o] + sum_{ky,kx,c} xp[n, oy*s+ky, ox*s+kx, c] w[o,ky,kx,c],
    xp = x zero-padded by `pad` on each spatial side."""
    N, H, W, C = x.shape
    O, KH, KW, _ = w.shape
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    OH = (H + 2 * pad - KH) // stride + 1
    OW = (W + 2 * pad - KW) // stride + 1
    y = np.zeros((N, OH, OW, O))
    for ky in range(KH):
        for kx in range(KW):
            patch = xp[:, ky:ky + stride * (OH - 1) + 1:stride, kx:kx + stride * (OW - 1) + 1:stride, :]
            y += patch @ w[:, ky, kx, :].T
    return y + b


def conv2d_backward(x, w, dy, stride, pad, need_dx=True):
    """Gradients of conv2d: dw[o,ky,kx,c] = sum dy[n,oy,ox,o] xp[n,oy*s+ky,ox*s+kx,c];
    db = sum dy; dxp[n,oy*s+ky,ox*s+kx,c] += sum_o dy w[o,ky,kx,c]."""
    N, H, W, C = x.shape
    O, KH, KW, _ = w.shape
    xp = np.pad(x, ((0, 0), (pad, pad), (pad, pad), (0, 0)))
    _, OH, OW, _ = dy.shape
    dw = np.zeros_like(w)
    dxp = np.zeros_like(xp) if need_dx else None
    dyf = dy.reshape(-1, O)
    for ky in range(KH):
        for kx in range(KW):
            sl = (slice(None), slice(ky, ky + stride * (OH - 1) + 1, stride),
                  slice(kx, kx + stride * (OW - 1) + 1, stride), slice(None))
            dw[:, ky, kx, :] = dyf.T @ xp[sl].reshape(-1, C)
            if need_dx:
                dxp[sl] += dy @ w[:, ky, kx, :]
    db = dyf.sum(axis=0)
    dx = None
    if need_dx:
        dx = dxp[:, pad:pad + H, pad:pad + W, :]
    return dx, dw, db


def maxpool_same(x, k=3, s=2):
    """TF 'same' max-pool: out = ceil(n/s); total pad = max((out-1)s + k - n, 0),
    top/left gets floor(pad/2); padding acts as -inf.  Returns (y, argmax index
    into the window, first maximum in (ky,kx) row-major order)."""
    N, H, W, C = x.shape
    OH, OW = _same_out(H, s), _same_out(W, s)
    ph = max((OH - 1) * s + k - H, 0)
    pw = max((OW - 1) * s + k - W, 0)
    xp = np.pad(x, ((0, 0), (ph // 2, ph - ph // 2), (pw // 2, pw - pw // 2), (0, 0)),
                constant_values=-np.inf)
    windows = np.stack([xp[:, ky:ky + s * (OH - 1) + 1:s, kx:kx + s * (OW - 1) + 1:s, :]
                        for ky in range(k) for kx in range(k)], axis=0)
    arg = np.argmax(windows, axis=0)          # first max in (ky,kx) order
    y = np.take_along_axis(windows, arg[None], axis=0)[0]
    return y, arg, (ph // 2, pw // 2)


def maxpool_same_backward(x_shape, arg, offs, dy, k=3, s=2):
    N, H, W, C = x_shape
    _, OH, OW, _ = dy.shape
    dx = np.zeros(x_shape)
    ky, kx = arg // k, arg % k
    n, oy, ox, c = np.meshgrid(np.arange(N), np.arange(OH), np.arange(OW), np.arange(C),
                               indexing="ij")
    iy = oy * s + ky - offs[0]
    ix = ox * s + kx - offs[1]
    np.add.at(dx, (n, iy, ix, c), dy)
    return dx


# ---- torsos ---------------------------------------------------------------
def torso_forward(spec, P, obs, emu=False):
    """obs [N][H][W][C] uint8 (or [N][D] float for the MLP).  Returns (features, cache).
    emu: bf16 weights and stored activations (C26); the MLP is fp32 on the GPU."""
    if spec.kind == NET_MLP:
        x = np.asarray(obs, np.float64).reshape(obs.shape[0], -1)
        cache = {"x0": x}
        for i in range(len(spec.mlp_hidden)):
            x = relu(x @ P[f"mlp{i}.w"].T + P[f"mlp{i}.b"])
            cache[f"x{i + 1}"] = x
        return x, cache
    x = np.asarray(obs, np.float64) / 255.0
    cache = {"x0": x}
    q = lambda t: _q(t, emu)
    if spec.kind == NET_ATARI_SHALLOW:
        a1 = q(relu(conv2d(x, q(P["conv1.w"]), P["conv1.b"], 4, 0)))
        a2 = q(relu(conv2d(a1, q(P["conv2.w"]), P["conv2.b"], 2, 0)))
        cache.update(a1=a1, a2=a2)
        flat = a2.reshape(a2.shape[0], -1)
    else:
        h = x
        for s in range(len(spec.sections)):
            conv = q(conv2d(h, q(P[f"s{s}.conv.w"]), P[f"s{s}.conv.b"], 1, 1))
            pooled, arg, offs = maxpool_same(conv)
            cache[f"s{s}.in"], cache[f"s{s}.conv"] = h, conv
            cache[f"s{s}.arg"], cache[f"s{s}.offs"] = arg, offs
            h = pooled
            for r in range(2):
                u0 = relu(h)
                t0 = conv2d(u0, q(P[f"s{s}.res{r}.conv0.w"]), P[f"s{s}.res{r}.conv0.b"], 1, 1)
                u1 = q(relu(t0))
                t1 = conv2d(u1, q(P[f"s{s}.res{r}.conv1.w"]), P[f"s{s}.res{r}.conv1.b"], 1, 1)
                cache[f"s{s}.res{r}"] = (h, u0, t0, u1)
                h = q(h + t1)
        cache["torso_pre"] = h
        flat = relu(h).reshape(h.shape[0], -1)
    fc = q(relu(flat @ q(P["fc.w"]).T + P["fc.b"]))
    cache.update(flat=flat, fc=fc)
    return fc, cache


def torso_backward(spec, P, cache, dfeat, grads, emu=False):
    """Backprop from d(features) into grads (dict); no gradient into obs.
    emu: bf16 weights in the data-gradient products and bf16-stored gradients."""
    if spec.kind == NET_MLP:
        d = dfeat
        for i in reversed(range(len(spec.mlp_hidden))):
            d = d * (cache[f"x{i + 1}"] > 0)
            grads[f"mlp{i}.w"] = d.T @ cache[f"x{i}"]
            grads[f"mlp{i}.b"] = d.sum(axis=0)
            d = d @ P[f"mlp{i}.w"]
        return
    q = lambda t: _q(t, emu)
    dfc = q(dfeat * (cache["fc"] > 0))
    grads["fc.w"] = dfc.T @ cache["flat"]
    grads["fc.b"] = dfc.sum(axis=0)
    dflat = dfc @ q(P["fc.w"])
    if spec.kind == NET_ATARI_SHALLOW:
        a1, a2 = cache["a1"], cache["a2"]
        da2 = q(dflat.reshape(a2.shape) * (a2 > 0))
        da1, grads["conv2.w"], grads["conv2.b"] = conv2d_backward(a1, q(P["conv2.w"]), da2, 2, 0)
        da1 = q(da1 * (a1 > 0))
        _, grads["conv1.w"], grads["conv1.b"] = conv2d_backward(cache["x0"], P["conv1.w"], da1,
                                                                4, 0, need_dx=False)
        return
    h_pre = cache["torso_pre"]
    dh = q(dflat.reshape(h_pre.shape) * (h_pre > 0))
    for s in reversed(range(len(spec.sections))):
        for r in reversed(range(2)):
            h_in, u0, t0, u1 = cache[f"s{s}.res{r}"]
            du1, grads[f"s{s}.res{r}.conv1.w"], grads[f"s{s}.res{r}.conv1.b"] = \
                conv2d_backward(u1, q(P[f"s{s}.res{r}.conv1.w"]), dh, 1, 1)
            dt0 = q(du1 * (t0 > 0))
            du0, grads[f"s{s}.res{r}.conv0.w"], grads[f"s{s}.res{r}.conv0.b"] = \
                conv2d_backward(u0, q(P[f"s{s}.res{r}.conv0.w"]), dt0, 1, 1)
            dh = q(dh + du0 * (h_in > 0))
        conv = cache[f"s{s}.conv"]
        dconv = q(maxpool_same_backward(conv.shape, cache[f"s{s}.arg"], cache[f"s{s}.offs"], dh))
        dh, grads[f"s{s}.conv.w"], grads[f"s{s}.conv.b"] = conv2d_backward(
            cache[f"s{s}.in"], q(P[f"s{s}.conv.w"]), dconv, 1, 1, need_dx=(s > 0))
        if dh is not None:
            dh = q(dh)


# ---- LSTM core (H3, H8; P:591 inputs, S:47/S:57 reset, C15) ----------------
def core_inputs(spec, fc, prev_action, reward, done, emu=False):
    """x_t = [fc_t, onehot(prev_a_t), clip(r_t, -1, 1)], one-hot and reward
    zeroed when done_t (C15); prev_action < 0 means 'none' (zero one-hot)."""
    A = spec.num_actions
    n = fc.shape[0]
    pa = np.asarray(prev_action).reshape(n).astype(np.int64)
    d = np.asarray(done).reshape(n).astype(bool)
    oh = np.zeros((n, A))
    ok = (pa >= 0) & (pa < A) & ~d
    oh[np.nonzero(ok)[0], pa[ok]] = 1.0
    r = np.clip(np.asarray(reward, np.float64).reshape(n), -1.0, 1.0) * (~d)
    return np.concatenate([fc, oh, _q(r, emu)[:, None]], axis=1)


def lstm_forward(P, X, done, h0, c0, emu=False):
    """X [B][T1][K] core inputs, done [B][T1], h0/c0 [B][U].  Gate order [i,f,g,o].
    for t: if done_t: (h,c) <- 0; z = Wx x_t + Wh h + b; c = f c + i g; h = o tanh c."""
    B, T1, _ = X.shape
    U = P["lstm.wh"].shape[1]
    h = np.asarray(h0, np.float64).copy()
    c = np.asarray(c0, np.float64).copy()
    d = np.asarray(done).astype(bool)
    H = np.zeros((B, T1, U))
    cache = dict(hprev=np.zeros((B, T1, U)), cprev=np.zeros((B, T1, U)),
                 gates=np.zeros((B, T1, 4 * U)), c=np.zeros((B, T1, U)))
    for t in range(T1):
        h = np.where(d[:, t, None], 0.0, h)
        c = np.where(d[:, t, None], 0.0, c)
        cache["hprev"][:, t], cache["cprev"][:, t] = h, c
        z = X[:, t] @ _q(P["lstm.wx"], emu).T + _q(h, emu) @ _q(P["lstm.wh"], emu).T + P["lstm.b"]
        i, f, g, o = (sigmoid(z[:, :U]), sigmoid(z[:, U:2 * U]), np.tanh(z[:, 2 * U:3 * U]),
                      sigmoid(z[:, 3 * U:]))
        c = f * c + i * g
        h = o * np.tanh(c)
        cache["gates"][:, t] = np.concatenate([i, f, g, o], axis=1)
        cache["c"][:, t] = c
        H[:, t] = h
    return H, cache


def lstm_backward(P, X, done, cache, dH, grads, emu=False):
    """BPTT through lstm_forward; returns dX.  No gradient into h0/c0.
    emu: dz rounded to bf16 for every product it enters (C26)."""
    B, T1, K = X.shape
    U = P["lstm.wh"].shape[1]
    d = np.asarray(done).astype(bool)
    dX = np.zeros_like(X)
    dWx = np.zeros_like(P["lstm.wx"])
    dWh = np.zeros_like(P["lstm.wh"])
    db = np.zeros_like(P["lstm.b"])
    dh_next = np.zeros((B, U))
    dc_next = np.zeros((B, U))
    for t in range(T1 - 1, -1, -1):
        gates = cache["gates"][:, t]
        i, f, g, o = gates[:, :U], gates[:, U:2 * U], gates[:, 2 * U:3 * U], gates[:, 3 * U:]
        c = cache["c"][:, t]
        cp = cache["cprev"][:, t]
        tc = np.tanh(c)
        dh = dH[:, t] + dh_next
        dc = dc_next + dh * o * (1.0 - tc ** 2)
        dz = np.concatenate([dc * g * i * (1 - i), dc * cp * f * (1 - f),
                             dc * i * (1 - g ** 2), dh * tc * o * (1 - o)], axis=1)
        dzq = _q(dz, emu)
        dWx += dzq.T @ X[:, t]
        dWh += dzq.T @ _q(cache["hprev"][:, t], emu)
        db += dzq.sum(axis=0)
        dX[:, t] = dzq @ _q(P["lstm.wx"], emu)
        dh_prev = dzq @ _q(P["lstm.wh"], emu)
        dc_prev = dc * f
        # the state entering step t was zeroed when done_t: no gradient flows past it
        dh_next = np.where(d[:, t, None], 0.0, dh_prev)
        dc_next = np.where(d[:, t, None], 0.0, dc_prev)
    grads["lstm.wx"], grads["lstm.wh"], grads["lstm.b"] = dWx, dWh, db
    return dX


# ---- whole network over a [B][T+1] batch ----------------------------------
def network_forward(spec, P, batch, emu=False):
    """Returns logits [B][T1][A], values [B][T1] and a cache for backward."""
    obs = batch["obs"]
    B, T1 = obs.shape[:2]
    frames = np.asarray(obs).reshape((B * T1,) + tuple(obs.shape[2:]))
    feat, tcache = torso_forward(spec, P, frames, emu)
    cache = dict(torso=tcache, B=B, T1=T1, emu=emu)
    if spec.lstm_units > 0:
        X = core_inputs(spec, feat, batch["prev_action"], batch["reward"], batch["done"], emu)
        X = X.reshape(B, T1, -1)
        H, lcache = lstm_forward(P, X, batch["done"], batch["h0"], batch["c0"], emu)
        cache.update(X=X, lstm=lcache)
        Hf = H.reshape(B * T1, -1)
    else:
        Hf = feat
    cache["H"] = Hf
    out = Hf @ P["heads.w"].T + P["heads.b"]
    A = spec.num_actions
    return out[:, :A].reshape(B, T1, A), out[:, A].reshape(B, T1), cache


def network_backward(spec, P, batch, cache, dlogits, dvalues):
    B, T1 = cache["B"], cache["T1"]
    A = spec.num_actions
    dout = np.concatenate([dlogits.reshape(B * T1, A), dvalues.reshape(B * T1, 1)], axis=1)
    grads = {"heads.w": dout.T @ cache["H"], "heads.b": dout.sum(axis=0)}
    dH = dout @ P["heads.w"]
    emu = cache.get("emu", False)
    if spec.lstm_units > 0:
        dX = lstm_backward(P, cache["X"], batch["done"], cache["lstm"],
                           dH.reshape(B, T1, -1), grads, emu)
        dfeat = dX.reshape(B * T1, -1)[:, :256]
    else:
        dfeat = dH
    torso_backward(spec, P, cache["torso"], dfeat, grads, emu)
    return grads


# --------------------------------------------------------------------------
# Clip + Adam (H11): S:75-93; clip 40 (C11); beta=(.9,.999) (C12).
# --------------------------------------------------------------------------
def clip_adam(params, grads, m, v, step, hp):
    """Returns (params', m', v', step', grad_norm, applied).  A non-finite norm
    skips the update and leaves the version unchanged."""
    g = np.asarray(grads, np.float64)
    norm = math.sqrt(float(np.sum(g * g)))
    if not math.isfinite(norm):
        return params.copy(), m.copy(), v.copy(), step, norm, 0
    if norm > hp["max_grad_norm"]:
        g = g * (hp["max_grad_norm"] / norm)
    t = step + 1
    b1, b2 = hp["beta1"], hp["beta2"]
    m2 = b1 * m + (1 - b1) * g
    v2 = b2 * v + (1 - b2) * g * g
    mh = m2 / (1 - b1 ** t)
    vh = v2 / (1 - b2 ** t)
    p2 = params - hp["lr"] * mh / (np.sqrt(vh) + hp["eps"])
    return p2, m2, v2, t, norm, 1


def learner_step(spec, params, m, v, step, batch, hp, emu=False):
    """One full learner step (H1-H11) on one [B][T+1] batch; DP semantics (C20):
    a single process on the concatenated batch with loss_scale = 1/(N B T).
    emu: bf16 rounding at the tensor-core path's rounding points (C26)."""
    P = unflatten(spec, params)
    logits, values, cache = network_forward(spec, P, batch, emu)
    L = policy_loss(logits, values, batch["action"], batch["behaviour_logp"],
                    batch["reward"], batch["done"], hp)
    grads = network_backward(spec, P, batch, cache, L["dlogits"], L["dvalues"])
    gflat = flatten(spec, grads)
    p2, m2, v2, step2, norm, applied = clip_adam(np.asarray(params, np.float64), gflat,
                                                 np.asarray(m, np.float64),
                                                 np.asarray(v, np.float64), step, hp)
    return dict(logits=logits, values=values, loss=L, grads=gflat, params=p2, m=m2, v=v2,
                step=step2, grad_norm=norm, applied=applied)


# --------------------------------------------------------------------------
# Centralized inference (H12, H13): S:434-442, reading C15-C19.
# --------------------------------------------------------------------------
def sample_inverse_cdf(logits, u):
    """a = min{ j : u < CDF_j } with CDF of softmax(logits) (C18); A-1 if none."""
    p = np.exp(log_softmax(np.asarray(logits, np.float64)))
    cdf = np.cumsum(p, axis=-1)
    idx = (u[:, None] < cdf).argmax(axis=-1)
    none = ~(u[:, None] < cdf).any(axis=-1)
    idx[none] = p.shape[-1] - 1
    return idx


def _infer_net(spec, params, table_h, table_c, table_last_action, actor_ids, obs, reward, done,
               emu=False):
    """The network part of a batched inference step: the A+1 head outputs
    of each request and the new (h, c) rows of the state table."""
    P = unflatten(spec, params)
    ids = np.asarray(actor_ids).astype(np.int64)
    d = np.asarray(done).astype(bool)
    th, tc, tla = table_h.copy(), table_c.copy(), table_last_action.copy()
    feat, _ = torso_forward(spec, P, np.asarray(obs), emu)
    if spec.lstm_units > 0:
        X = core_inputs(spec, feat, tla[ids], reward, d, emu)
        h0 = np.where(d[:, None], 0.0, th[ids].astype(np.float64))
        c0 = np.where(d[:, None], 0.0, tc[ids].astype(np.float64))
        H, lc = lstm_forward(P, X[:, None, :], np.zeros((len(ids), 1), bool), h0, c0, emu)
        h1, c1 = H[:, 0], lc["c"][:, 0]
        th[ids], tc[ids] = h1, c1
        feat = h1
    return feat @ P["heads.w"].T + P["heads.b"], ids, th, tc, tla


def infer(spec, params, table_h, table_c, table_last_action, actor_ids, obs, reward, done,
          uniforms, emu=False):
    """One batched inference call.  Returns (action, behaviour_logp, logits, new table
    arrays).  Actors not in actor_ids are untouched."""
    out, ids, th, tc, tla = _infer_net(spec, params, table_h, table_c, table_last_action, actor_ids,
                                       obs, reward, done, emu)
    A = spec.num_actions
    logits = out[:, :A]
    a = sample_inverse_cdf(logits, np.asarray(uniforms, np.float64))
    blp = np.take_along_axis(log_softmax(logits), a[:, None], axis=1)[:, 0]
    tla[ids] = a
    return a, blp, logits, th, tc, tla


def infer_eps_greedy(spec, params, table_h, table_c, table_last_action, actor_ids, obs, reward, done,
                     uniforms2, n_actors, base=0.4, alpha=7.0, emu=False):
    """R2D2 actors (P:591 dueling heads, P:614 per-actor epsilon-greedy): the same
    network step, Q from the A+1 outputs (dueling_q), the action epsilon-greedy with
    epsilon of the request's actor (table row).  Returns (action, behaviour_logp, Q,
    new table arrays)."""
    out, ids, th, tc, tla = _infer_net(spec, params, table_h, table_c, table_last_action, actor_ids,
                                       obs, reward, done, emu)
    A = spec.num_actions
    q = dueling_q(out[:, :A], out[:, A])
    u = np.asarray(uniforms2, np.float64)
    acts, blp = [], []
    for r, i in enumerate(ids):
        a, p = eps_greedy_action(q[r], actor_epsilon(int(i), n_actors, base, alpha), u[r, 0], u[r, 1])
        acts.append(a)
        blp.append(np.log(p))
    a = np.asarray(acts, np.int64)
    tla[ids] = a
    return a, np.asarray(blp), q, th, tc, tla


@dataclass
class UnrollStore:
    """Oracle of the device unroll store (C17, C19): per actor two (T+1)-slot
    buffers; slot T of unroll k is copied to slot 0 of unroll k+1."""
    T: int
    num_actors: int
    fill: np.ndarray = None
    cur: np.ndarray = None
    steps: dict = field(default_factory=dict)
    ready: list = field(default_factory=list)

    def __post_init__(self):
        self.fill = np.zeros(self.num_actors, np.int64)
        self.cur = np.zeros(self.num_actors, np.int64)

    def record(self, actor, step_record, h_before, c_before):
        key = (actor, int(self.cur[actor]))
        if self.fill[actor] == 0:
            self.steps[key] = dict(slots=[], h0=np.array(h_before), c0=np.array(c_before))
        self.steps[key]["slots"].append(step_record)
        self.fill[actor] += 1
        if self.fill[actor] == self.T + 1:
            self.ready.append(key)
            nxt = (actor, 1 - int(self.cur[actor]))
            self.steps[nxt] = dict(slots=[step_record], h0=np.array(h_before),
                                   c0=np.array(c_before))
            self.cur[actor] = 1 - self.cur[actor]
            self.fill[actor] = 1


# --------------------------------------------------------------------------
# Counter-based sampling stream (C18): Philox4x32-10 (Salmon et al., SC'11,
# the Random123 generator), keyed (seed) with counter (counter, actor id).
# --------------------------------------------------------------------------
_PHILOX_M = (0xD2511F53, 0xCD9E8D57)
_PHILOX_W = (0x9E3779B9, 0xBB67AE85)


def philox4x32_10(ctr, key):
    """ctr: 4 uint32 (arrays broadcast), key: 2 uint32.  10 rounds, key bumped
    between rounds: out = {hi1^c1^k0, lo1, hi0^c3^k1, lo0}."""
    c = [np.asarray(x, np.uint64) & 0xFFFFFFFF for x in ctr]
    k = [np.asarray(x, np.uint64) & 0xFFFFFFFF for x in key]
    for r in range(10):
        if r:
            k = [(k[0] + _PHILOX_W[0]) & 0xFFFFFFFF, (k[1] + _PHILOX_W[1]) & 0xFFFFFFFF]
        p0 = c[0] * _PHILOX_M[0]
        p1 = c[2] * _PHILOX_M[1]
        hi0, lo0 = p0 >> 32, p0 & 0xFFFFFFFF
        hi1, lo1 = p1 >> 32, p1 & 0xFFFFFFFF
        c = [hi1 ^ c[1] ^ k[0], lo1, hi0 ^ c[3] ^ k[1], lo0]
    return [x.astype(np.uint32) for x in c]


def philox_uniforms(seed, counter, actor_ids):
    """u = (x0 >> 8) * 2^-24 with x = Philox4x32-10(ctr = (counter lo, counter hi,
    actor id, 0), key = (seed lo, seed hi)) — one uniform per actor."""
    ids = np.asarray(actor_ids, np.uint64)
    x = philox4x32_10([counter & 0xFFFFFFFF, counter >> 32, ids, 0],
                      [seed & 0xFFFFFFFF, seed >> 32])
    return (x[0] >> 8).astype(np.float64) * (1.0 / 16777216.0)


# --------------------------------------------------------------------------
# R2D2 on SEED (hyper-parameters table
# `r2d2_params` P:586-622; SPEC qlearn S:187-245 and replay S:287-333).
# --------------------------------------------------------------------------
def value_rescale(x, eps=1e-3):
    """h(x) = sign(x)(sqrt(|x| + 1) - 1) + eps x (value function rescaling)."""
    x = np.asarray(x, np.float64)
    return np.sign(x) * (np.sqrt(np.abs(x) + 1.0) - 1.0) + eps * x


def value_rescale_inv(y, eps=1e-3):
    """h^-1(y) = sign(y)(((sqrt(1 + 4 eps (|y| + 1 + eps)) - 1) / (2 eps))^2 - 1) (S:204,
    the closed-form inverse of P:611's h)."""
    y = np.asarray(y, np.float64)
    return np.sign(y) * (((np.sqrt(1.0 + 4.0 * eps * (np.abs(y) + 1.0 + eps)) - 1.0) /
                          (2.0 * eps)) ** 2 - 1.0)


def r2d2_targets(q_online, q_target, actions, rewards, discounts, n=5, eta=0.9, eps=1e-3):
    """n-step double-Q targets with value rescaling and sequence priorities
    (P:149 double Q-learning, multi-step targets, value rescaling; P:613 n = 5;
    P:615 p = eta max_i delta_i + (1 - eta) mean delta).

    q_online, q_target: [B][T+1][A] rescaled action values of the online / target
    network at the T+1 observations of the trained part (after burn-in);
    actions [B][T+1] (a_t taken at observation t), rewards [B][T] (r_t received
    after a_t), discounts [B][T] (gamma_t = gamma (1 - done_{t+1}), the V-trace
    convention C5).  For t = 0..T-1, with m = min(n, T - t) (reading C32: the
    sequence end shortens the window; an episode end inside it zeroes the rest
    through gamma_t = 0):
      a* = argmax_a q_online[t+m][a]            (double Q: online selects, first max)
      G  = sum_{k<m} (prod_{j<k} gamma_{t+j}) r_{t+k}
           + (prod_{j<m} gamma_{t+j}) h^-1(q_target[t+m][a*])
      y_t = h(G);  delta_t = y_t - q_online[t][a_t]
    priority_b = eta max_t |delta_t| + (1 - eta) mean_t |delta_t|.
    Returns (y [B][T], delta [B][T], priority [B])."""
    qo = np.asarray(q_online, np.float64)
    qt = np.asarray(q_target, np.float64)
    a = np.asarray(actions).astype(np.int64)
    r = np.asarray(rewards, np.float64)
    g = np.asarray(discounts, np.float64)
    B, T = r.shape
    y = np.zeros((B, T))
    for b in range(B):
        for t in range(T):
            m = min(n, T - t)
            G, disc = 0.0, 1.0
            for k in range(m):
                G += disc * r[b, t + k]
                disc *= g[b, t + k]
            astar = int(np.argmax(qo[b, t + m]))
            G += disc * value_rescale_inv(qt[b, t + m, astar], eps)
            y[b, t] = value_rescale(G, eps)
    q_taken = np.take_along_axis(qo[:, :T], a[:, :T, None], axis=2)[:, :, 0]
    delta = y - q_taken
    ad = np.abs(delta)
    prio = eta * ad.max(axis=1) + (1.0 - eta) * ad.mean(axis=1)
    return y, delta, prio


def r2d2_loss_grad(q_online, actions, y, is_weights, scale):
    """L = scale sum_b w_b sum_t 1/2 (q_online[t][a_t] - y_t)^2 with y a constant
    (importance-weighted squared TD error); dL/dq_online is nonzero only at
    a_t: scale w_b (q - y).  Returns (loss, dq [B][T+1][A], row T zero)."""
    qo = np.asarray(q_online, np.float64)
    a = np.asarray(actions).astype(np.int64)
    B, T1, A = qo.shape
    T = T1 - 1
    w = np.asarray(is_weights, np.float64)
    dq = np.zeros_like(qo)
    loss = 0.0
    for b in range(B):
        for t in range(T):
            d = qo[b, t, a[b, t]] - y[b, t]
            loss += scale * w[b] * 0.5 * d * d
            dq[b, t, a[b, t]] = scale * w[b] * d
    return loss, dq


def replay_probabilities(priorities, alpha=0.9):
    """P(i) = p_i^alpha / sum_j p_j^alpha (P:602 priority exponent)."""
    p = np.asarray(priorities, np.float64) ** alpha
    return p / p.sum()


def replay_sample(priorities, uniforms, alpha=0.9, beta=0.6, size=None):
    """Proportional prioritized sampling by inverse CDF (the sum-tree's definition):
    draw i = min{ i : u * sum_j p_j^alpha < sum_{j<=i} p_j^alpha } for each uniform
    u in [0, 1); importance weights w_i = (N P(i))^-beta / max_batch w (P:603
    exponent 0.6; S:313, S:325 normalisation by the batch max), N = number of
    stored sequences (`size`, default len(priorities))."""
    pa = np.asarray(priorities, np.float64) ** alpha
    c = np.cumsum(pa)
    u = np.asarray(uniforms, np.float64)
    idx = np.searchsorted(c, u * c[-1], side="right")
    idx = np.minimum(idx, len(pa) - 1)
    N = len(pa) if size is None else size
    P = pa[idx] / c[-1]
    w = (N * P) ** (-beta)
    return idx, w / w.max()


def dueling_q(logits, values):
    """Dueling heads ("dueling heads"): Q(a) = V + A_a - mean_j A_j, with the
    net's A+1 outputs read as A advantages and 1 value (reading C35)."""
    adv = np.asarray(logits, np.float64)
    return np.asarray(values, np.float64)[..., None] + adv - adv.mean(axis=-1, keepdims=True)


def actor_epsilon(i, n_actors, base=0.4, alpha=7.0):
    """the i-th of N actors explores with epsilon_i = 0.4^(1 + 7 i / (N - 1))."""
    if n_actors <= 1:
        return float(base)
    return float(base) ** (1.0 + float(alpha) * i / (n_actors - 1))


def eps_greedy_action(q, eps, u_explore, u_action):
    """Epsilon-greedy over Q: with probability eps a uniformly random action
    (floor(u_action * A)), else the greedy one (first maximum); returns the action and
    its behaviour probability eps / A + (1 - eps) [a = greedy]."""
    q = np.asarray(q, np.float64)
    A = q.shape[-1]
    greedy = int(np.argmax(q))
    a = min(int(np.floor(u_action * A)), A - 1) if u_explore < eps else greedy
    return a, eps / A + ((1.0 - eps) if a == greedy else 0.0)


def r2d2_warm_state(spec, P, burn, emu=False):
    """Burn-in: run the network over the sequence's first burn_in steps from
    the stored state; the state entering the trained window (no gradient)."""
    _, _, cache = network_forward(spec, P, burn, emu)
    B, T1 = cache["B"], cache["T1"]
    H = cache["H"].reshape(B, T1, -1)
    return H[:, -1].copy(), cache["lstm"]["c"][:, -1].copy()


def r2d2_learner_step(spec, params, target_params, m, v, step, burn, train, is_weights, hp,
                      emu=False):
    """One R2D2 learner update: burn-in of the
    stored state by the online and the target network (no gradient), forward of the
    trained window [B][T+1] by both, dueling Q, n-step double-Q targets with value
    rescaling and priorities (r2d2_targets; trained step t uses reward[t+1] and
    gamma (1 - done[t+1]), C5), the IS-weighted squared-TD loss, its gradient through
    the dueling heads and the online network, clip + Adam.
    hp: dict(discount, n, eta, rescale_eps, loss_scale, lr, beta1, beta2, eps,
    max_grad_norm).  burn: None when burn_in = 0 (train's h0 / c0 are used)."""
    P = unflatten(spec, params)
    Pt = unflatten(spec, target_params)
    tr_o, tr_t = dict(train), dict(train)
    if burn is not None:
        tr_o["h0"], tr_o["c0"] = r2d2_warm_state(spec, P, burn, emu)
        tr_t["h0"], tr_t["c0"] = r2d2_warm_state(spec, Pt, burn, emu)
    lo, vo, cache = network_forward(spec, P, tr_o, emu)
    lt, vt, _ = network_forward(spec, Pt, tr_t, emu)
    qo, qt = dueling_q(lo, vo), dueling_q(lt, vt)
    rew = np.asarray(train["reward"], np.float64)[:, 1:]
    disc = hp["discount"] * (1.0 - np.asarray(train["done"], np.float64)[:, 1:])
    y, delta, prio = r2d2_targets(qo, qt, train["action"], rew, disc, hp["n"], hp["eta"],
                                  hp["rescale_eps"])
    w = np.ones(qo.shape[0]) if is_weights is None else np.asarray(is_weights, np.float64)
    loss, dq = r2d2_loss_grad(qo, train["action"], y, w, hp["loss_scale"])
    dA = dq - dq.sum(axis=-1, keepdims=True) / dq.shape[-1]
    dV = dq.sum(axis=-1)
    grads = network_backward(spec, P, tr_o, cache, dA, dV)
    gflat = flatten(spec, grads)
    p2, m2, v2, step2, norm, applied = clip_adam(np.asarray(params, np.float64), gflat,
                                                 np.asarray(m, np.float64),
                                                 np.asarray(v, np.float64), step, hp)
    return dict(q_online=qo, q_target=qt, y=y, delta=delta, priorities=prio, loss=loss,
                grads=gflat, params=p2, m=m2, v=v2, step=step2, grad_norm=norm, applied=applied,
                warm=(tr_o.get("h0"), tr_o.get("c0")))
