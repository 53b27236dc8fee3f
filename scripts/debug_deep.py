"""Stage-by-stage check of the c3 deep torso against the (emulated) oracle."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import seedgen
import paper_1910_06591_b200 as S

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
B, T = 2, 3
spec = S.spec_for_config(cfg)
ospec = {"c3": O.spec_c3, "c4": O.spec_c4}[cfg]()
params = seedgen.glorot_params(O.param_layout(ospec), seed=21, bias_std=0.1)
batch = seedgen.learner_batch((ospec.obs_h, ospec.obs_w, ospec.obs_c), ospec.num_actions, B, T,
                              seed=22, done_p=0.2, smm=(cfg == "c4"))
hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3)
L = S.Learner(spec, T, B, params, hp)
L.step({k: torch.from_numpy(v).cuda() for k, v in batch.items()})
torch.cuda.synchronize()
F_ = B * (T + 1)
P = O.unflatten(ospec, params)
frames = batch["obs"].reshape((F_,) + batch["obs"].shape[2:])
feat, cache = O.torso_forward(ospec, P, frames, emu=True)
def rel(a, b):
    return np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30)
H, W = ospec.obs_h, ospec.obs_w
for s, ch in enumerate(ospec.sections):
    H2, W2 = -(-H // 2), -(-W // 2)
    get = lambda n, shape: L.debug_buffer(f"s{s}.{n}", torch.bfloat16, shape).float().cpu().numpy()
    conv = get("conv", (F_, H, W, ch))
    print(f"s{s} conv", rel(conv, cache[f"s{s}.conv"]))
    h0 = get("h0", (F_, H2, W2, ch))
    hin0 = cache[f"s{s}.res0"][0]
    print(f"s{s} h0", rel(h0, hin0))
    arg = L.debug_buffer(f"s{s}.arg", torch.uint8, (F_, H2, W2, ch)).cpu().numpy()
    print(f"s{s} arg mismatch frac", np.mean(arg != cache[f"s{s}.arg"]))
    for r in range(2):
        u1 = get(f"u1{r}", (F_, H2, W2, ch))
        print(f"s{s} u1[{r}]", rel(u1, cache[f"s{s}.res{r}"][3]))
        hn = get(f"h{r+1}", (F_, H2, W2, ch))
        ref = cache[f"s{s}.res{r+1}"][0] if r == 0 else cache["torso_pre"] if s == len(ospec.sections) - 1 else None
        if ref is not None:
            print(f"s{s} h[{r+1}]", rel(hn, ref))
    H, W = H2, W2
# ---- backward ops on the GPU's own inputs
Pb = {k: O.bf16_round(v) for k, v in P.items()}
g = O.unflatten(ospec, L.grads.cpu().numpy().astype(np.float64))
nsec = len(ospec.sections)
s = nsec - 1
Hs, Ws = ospec.obs_h, ospec.obs_w
dims = []
for k in range(nsec):
    dims.append((Hs, Ws, -(-Hs // 2), -(-Ws // 2)))
    Hs, Ws = dims[-1][2], dims[-1][3]
H, W, H2, W2 = dims[s]
ch = ospec.sections[s]
bf = torch.bfloat16
dfc = L.debug_buffer("dfc", bf, (F_, 256)).float().cpu().numpy().astype(np.float64)
hr2 = L.debug_buffer(f"s{s}.hr2", bf, (F_, H2, W2, ch)).float().cpu().numpy().astype(np.float64)
dY2 = O.bf16_round((dfc @ Pb["fc.w"]).reshape(F_, H2, W2, ch) * (hr2 > 0))
q = O.bf16_round
getb = lambda n, shape: L.debug_buffer(f"s{s}.{n}", bf, shape).float().cpu().numpy().astype(np.float64)
dh = dY2
for r in (1, 0):
    u1 = getb(f"u1{r}", (F_, H2, W2, ch))
    hr = getb(f"hr{r}", (F_, H2, W2, ch))
    du1, dw1, db1 = O.conv2d_backward(u1, Pb[f"s{s}.res{r}.conv1.w"], dh, 1, 1)
    print(f"res{r}.conv1 wgrad", rel(g[f"s{s}.res{r}.conv1.w"], dw1), "bias", rel(g[f"s{s}.res{r}.conv1.b"], db1))
    dt0 = q(du1 * (u1 > 0))
    if r == 0:
        print("dt0[r=0]", rel(getb("dt0", (F_, H2, W2, ch)), dt0))
    du0, dw0, db0 = O.conv2d_backward(hr, Pb[f"s{s}.res{r}.conv0.w"], dt0, 1, 1)
    print(f"res{r}.conv0 wgrad", rel(g[f"s{s}.res{r}.conv0.w"], dw0), "bias", rel(g[f"s{s}.res{r}.conv0.b"], db0))
    dh = q(dh + du0 * (hr > 0))
print("dh(h0)", rel(getb("dhA", (F_, H2, W2, ch)), dh))
# ---- oracle's dfc / dh at the torso output vs the GPU's
hpo = hp.as_oracle()
logits, values, ocache = O.network_forward(ospec, P, batch, emu=True)
Lo = O.policy_loss(logits, values, batch["action"], batch["behaviour_logp"], batch["reward"], batch["done"], hpo)
dout = np.concatenate([Lo["dlogits"].reshape(F_, -1), Lo["dvalues"].reshape(F_, 1)], axis=1)
dH = dout @ P["heads.w"]
gr = {}
dX = O.lstm_backward(P, ocache["X"], batch["done"], ocache["lstm"], dH.reshape(B, T + 1, -1), gr, True)
dfeat = dX.reshape(F_, -1)[:, :256]
dfc_o = q(dfeat * (ocache["torso"]["fc"] > 0))
print("dfc gpu vs oracle", rel(dfc, dfc_o))
gl, gv = L.outputs()[0].cpu().numpy(), L.outputs()[1].cpu().numpy()
print("logits", rel(gl, logits), "values", rel(gv, values))
dl = L.debug_buffer("dlogits", torch.float32, (F_, ospec.num_actions)).cpu().numpy()
print("dlogits", rel(dl, Lo["dlogits"].reshape(F_, -1)))
dHg = L.debug_buffer("dH", torch.float32, (F_, 256)).cpu().numpy()
print("dH", rel(dHg, dH))
dG = L.debug_buffer("dG", bf, (F_, 1024)).float().cpu().numpy()
print("fc act gpu vs oracle", rel(L.debug_buffer("X", bf, (F_, 288)).float().cpu().numpy()[:, :256], ocache["torso"]["fc"]))
Pq = {k: q(v) for k, v in P.items()}
dflat_o = dfc_o @ Pq["fc.w"]
hpre_o = ocache["torso"]["torso_pre"]
dh_o = q(dflat_o.reshape(hpre_o.shape) * (hpre_o > 0))
print("dY2 gpu-derived vs oracle dh", rel(dY2, dh_o))
u1_o = ocache["torso"][f"s{s}.res1"][3]
_, dw_o, _ = O.conv2d_backward(u1_o, Pq[f"s{s}.res1.conv1.w"], dh_o, 1, 1)
ref_full = O.learner_step(ospec, params, np.zeros(params.size), np.zeros(params.size), 0, batch, hpo, emu=True)
gref = O.unflatten(ospec, ref_full["grads"])
print("oracle learner_step grad vs manual oracle", rel(gref[f"s{s}.res1.conv1.w"], dw_o))
print("gpu grad vs manual oracle", rel(g[f"s{s}.res1.conv1.w"], dw_o))
print("mask agreement", np.mean((hpre_o > 0) == (L.debug_buffer(f"s{s}.h2", bf, (F_, H2, W2, ch)).float().cpu().numpy() > 0)))
print("frac h_pre == 0 (oracle)", np.mean(hpre_o == 0), "frac |h|<1e-2", np.mean(np.abs(hpre_o) < 1e-2))
