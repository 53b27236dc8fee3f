"""GPU parity of seed_learner_step against the fp64 oracle (same seeded inputs).

Tolerances:
* fp32 paths (configs[0] MLP; V-trace/loss K2 given the network outputs):
  elementwise |gpu - ref| <= tol (|ref| + rms(ref)), tol = 1e-5 (V-trace) / 1e-4 (grads).
* bf16 tensor-core paths (configs[1] Atari net): per tensor
  ||gpu - ref||_2 / ||ref||_2 <= 2e-2 and max|gpu - ref| <= 2e-2 max|ref|.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle as O
import seedgen

pytestmark = pytest.mark.gpu


def _S():
    import paper_1910_06591_b200 as S
    return S


def scaled_check(gpu, ref, tol, what=""):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    rms = math.sqrt(float(np.mean(ref ** 2))) if ref.size else 0.0
    err = np.abs(gpu - ref)
    bound = tol * (np.abs(ref) + rms) + 1e-30
    worst = float(np.max(err / bound)) if ref.size else 0.0
    if os.environ.get("SEED_TEST_REPORT"):   # diagnostics: print every check, assert none
        print(f"CHECK {what} {worst:.3g} rel_l2 {np.linalg.norm(gpu - ref) / (np.linalg.norm(ref) + 1e-30):.3g}")
        return
    assert worst <= 1.0, f"{what}: worst err/bound = {worst:.3g}"


def bf16_check(gpu, ref, what="", tol=2e-2):
    gpu = np.asarray(gpu, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    nr = np.linalg.norm(ref)
    rel = np.linalg.norm(gpu - ref) / max(nr, 1e-30)
    mx = np.max(np.abs(gpu - ref)) / max(np.max(np.abs(ref)), 1e-30)
    assert rel <= tol and mx <= tol, f"{what}: relL2 {rel:.3g} max {mx:.3g}"
    return rel


def exact_bound_check(gpu, exact, emu, what="", floor=2e-2, factor=1.25):
    """Parity against the plain fp64 definition: the kernel may be no
    further from the exact oracle than bf16 rounding itself puts the oracle, i.e.
    ||gpu - exact|| / ||exact|| <= max(floor, factor * ||emu - exact|| / ||exact||)
    per tensor, where emu is the oracle taking its bf16 roundings at the kernels'
    rounding points (C26).  Returns (rel_gpu, rel_emu)."""
    gpu = np.asarray(gpu, np.float64).ravel()
    exact = np.asarray(exact, np.float64).ravel()
    emu = np.asarray(emu, np.float64).ravel()
    n = max(np.linalg.norm(exact), 1e-30)
    rg = np.linalg.norm(gpu - exact) / n
    re = np.linalg.norm(emu - exact) / n
    assert rg <= max(floor, factor * re), \
        f"{what}: gpu-vs-exact relL2 {rg:.3g} > max({floor}, {factor} x emu-vs-exact {re:.3g})"
    return rg, re


def _spec_pair(cfg):
    S = _S()
    spec = S.spec_for_config(cfg)
    ospec = {"c1": O.spec_c1, "c2": O.spec_c2, "c3": O.spec_c3, "c4": O.spec_c4,
             "c4m": O.spec_c4_medium, "c4l": O.spec_c4_large, "c3m": O.spec_c3_medium,
             "c3l": O.spec_c3_large}[cfg]()
    return spec, ospec


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c4m", "c4l", "c3m", "c3l"])
def test_param_layout_matches_oracle(cfg):
    S = _S()
    spec, ospec = _spec_pair(cfg)
    assert S.net_param_layout(spec) == [(n, tuple(s)) for n, s in O.param_layout(ospec)]
    assert S.net_param_count(spec) == O.param_count(ospec)


def _make(cfg, B, T, seed=0, done_p=0.05, force_done=(), hp_over=None):
    S = _S()
    spec, ospec = _spec_pair(cfg)
    layout = O.param_layout(ospec)
    params = seedgen.glorot_params(layout, seed=seed + 10, bias_std=0.1,
                                   lstm_units=max(ospec.lstm_units, 1))
    obs_shape = (ospec.obs_dim,) if cfg == "c1" else (ospec.obs_h, ospec.obs_w, ospec.obs_c)
    batch = seedgen.learner_batch(obs_shape, ospec.num_actions, B, T, seed=seed,
                                  lstm_units=ospec.lstm_units, done_p=done_p,
                                  float_obs=(cfg == "c1"), force_done=force_done)
    hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3)
    for k, v in (hp_over or {}).items():
        setattr(hp, k, v)
    return S, spec, ospec, params, batch, hp


def _gpu_batch(batch):
    out = {}
    for k, v in batch.items():
        out[k] = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    return out


def _run_gpu(S, spec, params, batch, hp, B, T, steps=1):
    L = S.Learner(spec, T, B, params, hp)
    gb = _gpu_batch(batch)
    for _ in range(steps):
        m = L.step(gb)
    torch.cuda.synchronize()
    logits, values, vs, pg = (x.cpu().numpy().astype(np.float64) for x in L.outputs())
    return dict(L=L, metrics=m.cpu().numpy(), logits=logits, values=values, vs=vs, pg=pg,
                grads=L.grads.cpu().numpy().astype(np.float64),
                params=L.params.cpu().numpy().astype(np.float64),
                m=L.m.cpu().numpy().astype(np.float64), v=L.v.cpu().numpy().astype(np.float64),
                step=int(L.step_counter.item()))


def _per_tensor(ospec, flat):
    return O.unflatten(ospec, flat)


def _check_k2_and_adam(ospec, params, batch, hp, g, tol=1e-5):
    """K2 (loss) and K9 (clip+Adam) checked tightly on the GPU's own inputs."""
    L = O.policy_loss(g["logits"], g["values"], batch["action"], batch["behaviour_logp"],
                      batch["reward"], batch["done"], hp.as_oracle())
    scaled_check(g["vs"], L["vs"], tol, "vs(K2)")
    scaled_check(g["pg"], L["pg_adv"], tol, "pg_adv(K2)")
    scaled_check(g["metrics"][1], L["pg"], 1e-4, "pg loss")
    scaled_check(g["metrics"][2], L["baseline"], 1e-4, "baseline loss")
    scaled_check(g["metrics"][3], L["entropy"], 1e-4, "entropy loss")
    p2, m2, v2, step2, norm, applied = O.clip_adam(
        params.astype(np.float64), g["grads"], np.zeros(params.size), np.zeros(params.size), 0,
        hp.as_oracle())
    assert applied == 1 and g["step"] == 1 and g["metrics"][5] == 1.0
    scaled_check(g["metrics"][4], norm, 1e-5, "grad norm")
    scaled_check(g["m"], m2, 1e-5, "adam m")
    scaled_check(g["v"], v2, 1e-5, "adam v")
    scaled_check(g["params"] - params, p2 - params, 1e-3, "adam update")
    return L


def test_learner_c1_mlp_fp32_parity():
    B, T = 8, 20
    S, spec, ospec, params, batch, hp = _make("c1", B, T, seed=1, done_p=0.1)
    g = _run_gpu(S, spec, params, batch, hp, B, T)
    ref = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0, batch,
                         hp.as_oracle())
    scaled_check(g["logits"], ref["logits"], 1e-5, "logits")
    scaled_check(g["values"], ref["values"], 1e-5, "values")
    scaled_check(g["vs"], ref["loss"]["vs"], 1e-5, "vs")
    scaled_check(g["pg"], ref["loss"]["pg_adv"], 1e-5, "pg_adv")
    gt, rt = _per_tensor(ospec, g["grads"]), _per_tensor(ospec, ref["grads"])
    for name, _ in O.param_layout(ospec):
        scaled_check(gt[name], rt[name], 1e-4, f"grad {name}")
    scaled_check(g["metrics"][0], ref["loss"]["loss"], 1e-5, "loss")
    scaled_check(g["params"] - params, ref["params"] - params, 1e-3, "update")
    _check_k2_and_adam(ospec, params, batch, hp, g)


@pytest.mark.parametrize("B,T,seed", [(4, 5, 0), (3, 7, 1), (32, 20, 2), (33, 4, 5)])
def test_learner_c2_atari_parity(B, T, seed):
    """C22 tolerance against the oracle taking the ReLU decisions in the kernels'
    (bf16) precision (C26); the exact-fp64 deviation is reported alongside."""
    S, spec, ospec, params, batch, hp = _make("c2", B, T, seed=seed, done_p=0.1,
                                              force_done=((0, 0), (1, T)))
    g = _run_gpu(S, spec, params, batch, hp, B, T)
    ref = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0, batch,
                         hp.as_oracle(), emu=True)
    exact = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0,
                           batch, hp.as_oracle())
    bf16_check(g["logits"], exact["logits"], "logits vs exact")
    bf16_check(g["values"], exact["values"], "values vs exact")
    ex = O.unflatten(ospec, exact["grads"])
    bf16_check(g["logits"], ref["logits"], "logits")
    bf16_check(g["values"], ref["values"], "values")
    bf16_check(g["vs"], ref["loss"]["vs"], "vs")
    bf16_check(g["pg"], ref["loss"]["pg_adv"], "pg_adv")
    gt, rt = _per_tensor(ospec, g["grads"]), _per_tensor(ospec, ref["grads"])
    errs = {}
    for name, _ in O.param_layout(ospec):
        try:
            errs[name] = f"{bf16_check(gt[name], rt[name], name):.2e}"
        except AssertionError as e:
            errs[name] = "FAIL " + str(e)
    print("per-tensor grad relL2 (vs emulated):", errs)
    assert not any(v.startswith("FAIL") for v in errs.values()), errs
    # every gradient tensor against the exact definition (C26, C31)
    ex_rel = {}
    for name, _ in O.param_layout(ospec):
        rg, re = exact_bound_check(gt[name], ex[name], rt[name], f"grad {name} vs exact")
        ex_rel[name] = f"{rg:.2e} (emu {re:.2e})"
    print("per-tensor grad relL2 vs exact, gpu (emu):", ex_rel)
    _check_k2_and_adam(ospec, params, batch, hp, g)


def test_learner_c2_multi_step_and_version():
    B, T = 4, 6
    S, spec, ospec, params, batch, hp = _make("c2", B, T, seed=3)
    g = _run_gpu(S, spec, params, batch, hp, B, T, steps=3)
    assert g["step"] == 3 and g["metrics"][6] == 3.0
    P = params.astype(np.float64)
    m = np.zeros(P.size)
    v = np.zeros(P.size)
    step = 0
    for _ in range(3):
        ref = O.learner_step(ospec, P, m, v, step, batch, hp.as_oracle(), emu=True)
        P, m, v, step = ref["params"], ref["m"], ref["v"], ref["step"]
    # Adam normalises each coordinate (update ~ lr * sign(g) where |g| ~ noise), so
    # only the tensor-level relative L2 is a well-conditioned criterion here.
    d_gpu, d_ref = g["params"] - params, P - params
    rel = np.linalg.norm(d_gpu - d_ref) / np.linalg.norm(d_ref)
    assert rel <= 2e-2, rel


def test_learner_nonfinite_skips_update():
    B, T = 4, 5
    S, spec, ospec, params, batch, hp = _make("c2", B, T, seed=4)
    batch["reward"][1, 3] = np.nan
    g = _run_gpu(S, spec, params, batch, hp, B, T)
    assert g["metrics"][5] == 0.0 and g["metrics"][7] == 1.0
    assert g["step"] == 0
    np.testing.assert_array_equal(g["params"], params.astype(np.float64))


def _deep_dims(ospec):
    H, W, out = ospec.obs_h, ospec.obs_w, []
    for ch in ospec.sections:
        out.append((H, W, -(-H // 2), -(-W // 2), ch))
        H, W = out[-1][2], out[-1][3]
    return out


def _padded_rows(L, name, shape):
    """Decode a deep-torso activation buffer (conv3w.cuh layout: rows of the padded
    (H+2) x (W+2) space, C bf16 channels per row, 16-byte chunks stored at the
    32B / 64B swizzled position) into dense (F, H, W, C) float64, and check that
    the border rows hold zeros."""
    F_, H, W, C = shape
    if C > 64:   # two planes of 64-channel rows (conv3w.cuh), concatenated on channels
        rows = F_ * (H + 2) * (W + 2)
        raw = L.debug_buffer(name, torch.uint8, (2, rows, 128)).cpu().numpy()
        planes = [_decode_rows(raw[q], shape[:3] + (64,), name) for q in range(2)]
        return np.concatenate(planes, axis=-1)
    rows, rb = F_ * (H + 2) * (W + 2), 2 * C
    raw = L.debug_buffer(name, torch.uint8, (rows, rb)).cpu().numpy()
    return _decode_rows(raw, shape, name)


def _decode_rows(raw, shape, name):
    F_, H, W, C = shape
    rows, rb = F_ * (H + 2) * (W + 2), 2 * C
    g = np.arange(rows)[:, None]
    j = np.arange(rb // 16)[None, :]
    phys = j ^ (((g >> 2) & 1) if rb == 32 else ((g >> 1) & 3) if rb == 64 else (g & 7))
    chunks = raw.reshape(rows, rb // 16, 16)
    dense = np.take_along_axis(chunks, phys[:, :, None], axis=1).reshape(rows, rb)
    v = torch.from_numpy(np.ascontiguousarray(dense)).view(torch.bfloat16).float().numpy()
    v = v.reshape(F_, H + 2, W + 2, C).astype(np.float64)
    border = v.copy()
    border[:, 1:-1, 1:-1, :] = 0
    if not name.endswith(".conv"):   # the section conv output's border is never read
        assert not np.any(border), f"{name}: nonzero border rows"
    return v[:, 1:-1, 1:-1, :]


@pytest.mark.parametrize("cfg,B,T", [("c3", 2, 3), ("c4", 2, 2), ("c3", 3, 1), ("c4m", 2, 2),
                                     ("c4l", 1, 2), ("c3m", 2, 3), ("c3l", 1, 1)])
def test_learner_deep_parity(cfg, B, T, monkeypatch):
    """configs[2] (DMLab IMPALA-deep, 72x96x3) / configs[3] (GRF SMM 72x96x16), full
    image size: 3x3 'same' convs, max-pool, residual blocks (C14).

    Forward: logits/values and every section's activations vs the emulated oracle
    (C22).  Backward: 15-20 stacked bf16 convs move activations by ~3e-3 and flip
    ~0.05% of the ReLU masks, which alone is a few % rel-L2 on torso gradients, so
    the torso backward is checked stage-wise: the oracle's backward of each section
    runs on the GPU's own activations and incoming gradient (teacher forcing) and
    every weight/bias gradient (5e-3 elementwise-scaled: fp32 reductions over up to
    F*H*W rows, and the incoming dh of a lower section is the oracle's re-rounded dgrad),
    dh and dconv must agree.
    FC / LSTM / heads gradients, V-trace, loss and Adam are checked end to end."""
    S = _S()
    spec, ospec = _spec_pair(cfg)
    params = seedgen.glorot_params(O.param_layout(ospec), seed=21, bias_std=0.1)
    batch = seedgen.learner_batch((ospec.obs_h, ospec.obs_w, ospec.obs_c), ospec.num_actions, B,
                                  T, seed=22, done_p=0.2, smm=cfg.startswith("c4"))
    hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3)
    # the fused section conv + max-pool (conv3w_pool.cu) keeps the conv output on
    # chip; this makes it also store the conv rows for the checks below
    monkeypatch.setenv("SEED_STORE_CONV", "1")
    g = _run_gpu(S, spec, params, batch, hp, B, T)
    L = g["L"]
    ref = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0, batch,
                         hp.as_oracle(), emu=True)
    bf16_check(g["logits"], ref["logits"], "logits")
    bf16_check(g["values"], ref["values"], "values")
    gt, rt = _per_tensor(ospec, g["grads"]), _per_tensor(ospec, ref["grads"])
    _check_k2_and_adam(ospec, params, batch, hp, g)
    # heads gradients on the GPU's own output gradients and LSTM outputs (fp32 path)
    Hh = L.debug_buffer("H", torch.float32, (B * (T + 1), 256)).cpu().numpy().astype(np.float64)
    dl = L.debug_buffer("dlogits", torch.float32, (B * (T + 1), ospec.num_actions)).cpu().numpy()
    dv = L.debug_buffer("dvalues", torch.float32, (B * (T + 1), 1)).cpu().numpy()
    dout = np.concatenate([dl, dv], axis=1).astype(np.float64)
    scaled_check(gt["heads.w"], dout.T @ Hh, 1e-4, "heads.w (teacher-forced)")
    scaled_check(gt["heads.b"], dout.sum(0), 1e-4, "heads.b (teacher-forced)")
    # LSTM weight gradients on the GPU's own dG, core input X and h_{t-1}
    F0 = B * (T + 1)
    Kx = 256 + ospec.num_actions + 1
    dG = L.debug_buffer("dG", torch.bfloat16, (F0, 1024)).float().cpu().numpy().astype(np.float64)
    Xg = L.debug_buffer("X", torch.bfloat16, (F0, -1)).float().cpu().numpy().astype(np.float64)
    Hp = L.debug_buffer("Hprev", torch.bfloat16, (F0, 256)).float().cpu().numpy().astype(np.float64)
    scaled_check(gt["lstm.wx"], dG.T @ Xg[:, :Kx], 1e-3, "lstm.wx (teacher-forced)")
    scaled_check(gt["lstm.b"], dG.sum(0), 1e-3, "lstm.b (teacher-forced)")
    scaled_check(gt["lstm.wh"], dG.T @ Hp, 1e-3, "lstm.wh (teacher-forced)")

    # ---- forward activations per section
    F_ = B * (T + 1)
    P = O.unflatten(ospec, params)
    frames = batch["obs"].reshape((F_,) + batch["obs"].shape[2:])
    _, cache = O.torso_forward(ospec, P, frames, emu=True)
    bf = torch.bfloat16
    dims = _deep_dims(ospec)

    def buf(s, n, shape):
        return _padded_rows(L, f"s{s}.{n}", shape)

    for s, (H, W, H2, W2, ch) in enumerate(dims):
        bf16_check(buf(s, "conv", (F_, H, W, ch)), cache[f"s{s}.conv"], f"s{s}.conv")
        for r in range(2):
            bf16_check(buf(s, f"u1{r}", (F_, H2, W2, ch)), cache[f"s{s}.res{r}"][3], f"s{s}.u1[{r}]")
    # ---- teacher-forced backward, section by section
    q = O.bf16_round
    Pq = {k: q(v) for k, v in P.items()}
    last = len(dims) - 1
    dfc = L.debug_buffer("dfc", bf, (F_, 256)).float().cpu().numpy().astype(np.float64)
    H, W, H2, W2, ch = dims[last]
    hr2 = buf(last, "hr2", (F_, H2, W2, ch))
    act2 = hr2.reshape(F_, -1)
    np.testing.assert_array_equal(
        L.debug_buffer("act2", bf, (F_, act2.shape[1])).float().cpu().numpy(), act2)
    scaled_check(gt["fc.w"], dfc.T @ act2, 1e-3, "fc.w (teacher-forced)")
    scaled_check(gt["fc.b"], dfc.sum(0), 1e-3, "fc.b (teacher-forced)")
    dh = q((dfc @ Pq["fc.w"]).reshape(F_, H2, W2, ch) * (hr2 > 0))
    # teacher-forced stage tolerance: the incoming dh of each block is the oracle's
    # re-rounded chain, whose drift from the kernel's own grows with the block width
    # (128-channel DMLab 4x: measured worst 1.32x of 5e-3 at rel-L2 4.6e-4, s1.res0.conv0)
    ttol = 5e-3 if max(ospec.sections) <= 64 else 1e-2
    for s in range(last, -1, -1):
        H, W, H2, W2, ch = dims[s]
        for r in (1, 0):
            u1 = buf(s, f"u1{r}", (F_, H2, W2, ch))
            hr = buf(s, f"hr{r}", (F_, H2, W2, ch))
            du1, dw1, db1 = O.conv2d_backward(u1, Pq[f"s{s}.res{r}.conv1.w"], dh, 1, 1)
            scaled_check(gt[f"s{s}.res{r}.conv1.w"], dw1, ttol, f"s{s}.res{r}.conv1.w")
            scaled_check(gt[f"s{s}.res{r}.conv1.b"], db1, ttol, f"s{s}.res{r}.conv1.b")
            dt0 = q(du1 * (u1 > 0))
            du0, dw0, db0 = O.conv2d_backward(hr, Pq[f"s{s}.res{r}.conv0.w"], dt0, 1, 1)
            scaled_check(gt[f"s{s}.res{r}.conv0.w"], dw0, ttol, f"s{s}.res{r}.conv0.w")
            scaled_check(gt[f"s{s}.res{r}.conv0.b"], db0, ttol, f"s{s}.res{r}.conv0.b")
            dh = q(dh + du0 * (hr > 0))
        bf16_check(buf(s, "dhA", (F_, H2, W2, ch)), dh, f"s{s}.dh(h0)", tol=1e-2)
        if ch > 64:   # two planes of 64 channels
            arg = L.debug_buffer(f"s{s}.arg", torch.uint8, (2, F_, H2 + 2, W2 + 2, 64)).cpu().numpy()
            arg = np.concatenate([arg[0], arg[1]], axis=-1)
        else:
            arg = L.debug_buffer(f"s{s}.arg", torch.uint8, (F_, H2 + 2, W2 + 2, ch)).cpu().numpy()
        arg = arg[:, 1:-1, 1:-1, :]
        # max-pool argmax is index work: bit-exact against the oracle's max-pool run on
        # the GPU's own conv output (first maximum in (ky, kx) order, -inf padding)
        gconv = buf(s, "conv", (F_, H, W, ch))
        ry, rarg, _ = O.maxpool_same(gconv)
        np.testing.assert_array_equal(arg.astype(np.int64), rarg, err_msg=f"s{s} pool argmax")
        np.testing.assert_array_equal(buf(s, "h0", (F_, H2, W2, ch)), ry,
                                      err_msg=f"s{s} pooled values")
        cin = ospec.obs_c if s == 0 else dims[s - 1][4]
        dconv = np.zeros((F_, H, W, ch))
        offs = ((max((H2 - 1) * 2 + 3 - H, 0)) // 2, (max((W2 - 1) * 2 + 3 - W, 0)) // 2)
        dconv = q(O.maxpool_same_backward((F_, H, W, ch), arg.astype(np.int64), offs,
                                          buf(s, "dhA", (F_, H2, W2, ch))))
        gd = buf(s, "dconv", (F_, H, W, ch))
        bf16_check(gd, dconv, f"s{s}.dconv", tol=1e-2)
        xin = (frames.astype(np.float64) / 255.0 if s == 0 else
               buf(s - 1, "h2", (F_, H, W, cin)))
        dxin, dw, db = O.conv2d_backward(xin, Pq[f"s{s}.conv.w"], gd, 1, 1, need_dx=(s > 0))
        scaled_check(gt[f"s{s}.conv.w"], dw, ttol, f"s{s}.conv.w")
        scaled_check(gt[f"s{s}.conv.b"], db, ttol, f"s{s}.conv.b")
        if s > 0:
            dh = q(dxin)
    # end to end, every gradient tensor against the exact fp64 definition (C31)
    exact = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0, batch,
                           hp.as_oracle())
    ex = O.unflatten(ospec, exact["grads"])
    _deep_exact_checks(cfg, g, gt, ex, rt, exact, ref)


def _deep_exact_checks(cfg, g, gt, ex, rt, exact, ref):
    """IMPALA-deep torsos (15-20 stacked bf16 convs, C31): the kernel and the emulated
    oracle are two bf16 evaluations whose ReLU-mask / argmax flips are different
    samples of the same rounding noise, so per tensor their distances to the exact
    definition agree only up to sampling spread (measured 0.7-1.3x at F = 202).
    Criterion: the whole gradient vector within 1.25x of the emulated oracle's
    distance, every tensor within 1.5x (floor 2e-2), logits / values within 1.25x."""
    allg = np.concatenate([np.ravel(gt[n]) for n in gt])
    alle = np.concatenate([np.ravel(ex[n]) for n in gt])
    allr = np.concatenate([np.ravel(rt[n]) for n in gt])
    rows, bad = {}, []
    try:
        rg, re = exact_bound_check(allg, alle, allr, "whole gradient")
        rows["(all)"] = f"{rg:.2e} (emu {re:.2e})"
    except AssertionError as e:
        bad.append(str(e))
    for n in gt:
        try:
            rg, re = exact_bound_check(gt[n], ex[n], rt[n], n, factor=1.5)
        except AssertionError as e:
            bad.append(str(e))
            rg = np.linalg.norm(gt[n] - ex[n]) / np.linalg.norm(ex[n])
            re = np.linalg.norm(rt[n] - ex[n]) / np.linalg.norm(ex[n])
        rows[n] = f"{rg:.2e} (emu {re:.2e})"
    for what in ("logits", "values"):
        try:
            exact_bound_check(g[what], exact[what], ref[what], what)
        except AssertionError as e:
            bad.append(str(e))
    print(cfg, "grad relL2 vs exact, gpu (emu):", rows)
    assert not bad, bad


@pytest.mark.parametrize("cfg,B,T", [("c3", 32, 100), ("c4", 128, 32), ("c4l", 128, 32),
                                     ("c3m", 32, 100), ("c3l", 32, 100)])
def test_learner_deep_full_size_sampled(cfg, B, T):
    """BASELINE.json configs[2] / configs[3] at their full sizes (the shapes bench.py
    times: F = 3232 / 4224 frames, 23-31 M padded rows at 72x96): one learner step,
    then the torso output of sampled frames (relu(h) of the last section, the FC
    input, and the FC output) against the emulated oracle run on those frames alone
    (C22), plus finite loss / gradients."""
    S = _S()
    spec, ospec = _spec_pair(cfg)
    params = seedgen.glorot_params(O.param_layout(ospec), seed=31, bias_std=0.1)
    batch = seedgen.learner_batch((ospec.obs_h, ospec.obs_w, ospec.obs_c), ospec.num_actions, B,
                                  T, seed=32, smm=cfg.startswith("c4"))
    hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-4)
    L = S.Learner(spec, T, B, params, hp)
    m = L.step(_gpu_batch(batch))
    torch.cuda.synchronize()
    assert np.all(np.isfinite(m.cpu().numpy()[:5])) and float(m[5].item()) == 1.0
    assert bool(torch.isfinite(L.grads).all())
    F_ = B * (T + 1)
    frames = batch["obs"].reshape((F_,) + batch["obs"].shape[2:])
    rng = np.random.default_rng(33)
    pick = np.sort(rng.choice(F_, 4, replace=False))
    pick[-1] = F_ - 1                       # the last frame (end of the row space)
    _, cache = O.torso_forward(ospec, O.unflatten(ospec, params), frames[pick], emu=True)
    bf = torch.bfloat16
    act2 = L.debug_buffer("act2", bf, (F_, -1)).float().cpu().numpy().astype(np.float64)
    bf16_check(act2[pick], cache["flat"], f"{cfg} torso output (sampled frames)")
    X = L.debug_buffer("X", bf, (F_, -1)).float().cpu().numpy().astype(np.float64)
    bf16_check(X[pick, :256], cache["fc"], f"{cfg} fc output (sampled frames)")


def test_learner_c3_bptt_T100():
    """configs[2] at its full unroll length T = 100 (101 serial LSTM steps forward and
    backward) and full image size, B = 2: logits, values and the LSTM / heads
    gradients against the emulated oracle (C22) and every gradient tensor end to end
    against the exact fp64 definition (C31).  One forced episode boundary mid-unroll
    (the BPTT chain is cut there), otherwise done ~ Bern(1/200)."""
    S = _S()
    B, T = 2, 100
    spec, ospec = _spec_pair("c3")
    params = seedgen.glorot_params(O.param_layout(ospec), seed=41, bias_std=0.1)
    batch = seedgen.learner_batch((ospec.obs_h, ospec.obs_w, ospec.obs_c), ospec.num_actions, B,
                                  T, seed=42, done_p=1.0 / 200, force_done=((1, 57),))
    hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3)
    g = _run_gpu(S, spec, params, batch, hp, B, T)
    z = np.zeros(params.size)
    ref = O.learner_step(ospec, params, z, z, 0, batch, hp.as_oracle(), emu=True)
    exact = O.learner_step(ospec, params, z, z, 0, batch, hp.as_oracle())
    bf16_check(g["logits"], ref["logits"], "logits")
    bf16_check(g["values"], ref["values"], "values")
    gt, rt = _per_tensor(ospec, g["grads"]), _per_tensor(ospec, ref["grads"])
    ex = O.unflatten(ospec, exact["grads"])
    for n in ("heads.w", "heads.b", "lstm.wx", "lstm.wh", "lstm.b"):
        bf16_check(gt[n], rt[n], f"{n} (T=100 BPTT)")
    _check_k2_and_adam(ospec, params, batch, hp, g)
    _deep_exact_checks("c3 T=100", g, gt, ex, rt, exact, ref)


def test_learner_c4_u8_source_parity(tmp_path):
    """The opt-in XF_U8 path (SEED_XF_U8=1: section 0 reads the uint8 obs and expands
    them to bf16 rows in shared memory, no obs_bf16 pass) and the unfused section
    conv + max-pool (SEED_FUSE_POOL=0) give the same learner step as the default
    path: logits / values and gradients within fp32 accumulation-order noise (run in
    subprocesses: the switches are read once)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O, seedgen, paper_1910_06591_b200 as S
B, T = 2, 3
spec = S.spec_for_config("c4")
params = seedgen.glorot_params(O.param_layout(O.spec_c4()), seed=21, bias_std=0.1)
batch = seedgen.learner_batch((72, 96, 16), 19, B, T, seed=22, done_p=0.2, smm=True)
L = S.Learner(spec, T, B, params, S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3))
L.step({k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in batch.items()})
torch.cuda.synchronize()
np.save(sys.argv[1], np.concatenate([L.outputs()[0].cpu().numpy().ravel(), L.grads.cpu().numpy()]))
''' % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    # default; XF_U8 section 0; every section conv + max-pool unfused (SEED_FUSE_POOL=0)
    for name, env in (("d", {}), ("u8", {"SEED_XF_U8": "1"}), ("nofuse", {"SEED_FUSE_POOL": "0"})):
        f = tmp_path / f"o_{name}.npy"
        subprocess.run([sys.executable, "-c", code, str(f)], check=True, timeout=300,
                       env=dict(os.environ, **env))
        outs.append(np.load(f).astype(np.float64))
    for o in outs[1:]:
        rel = np.linalg.norm(o - outs[0]) / np.linalg.norm(outs[0])
        assert rel < 1e-3, rel
