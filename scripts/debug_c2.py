"""Layer-by-layer check of the c2 backward using GPU intermediates as oracle inputs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle as O
import seedgen
import paper_1910_06591_b200 as S

B, T = 4, 5
spec = S.spec_for_config("c2"); ospec = O.spec_c2()
params = seedgen.glorot_params(O.param_layout(ospec), seed=10, bias_std=0.1)
batch = seedgen.learner_batch((84, 84, 4), 18, B, T, seed=0, done_p=0.1)
hp = S.HParams(lam=0.95, loss_scale=1.0 / (B * T), lr=1e-3)
L = S.Learner(spec, T, B, params, hp)
L.step({k: torch.from_numpy(v).cuda() for k, v in batch.items()})
torch.cuda.synchronize()
F = B * (T + 1)
bf = torch.bfloat16
get = lambda n, dt, sh: L.debug_buffer(n, dt, sh).float().cpu().numpy().astype(np.float64)
act1 = get("act1", bf, (F, 20, 20, 16)); act2 = get("act2", bf, (F, 9, 9, 32))
dY2 = get("dY2", bf, (F, 9, 9, 32)); dY1 = get("dY1", bf, (F, 20, 20, 16)); dfc = get("dfc", bf, (F, 256))
X = get("X", bf, (F, 288)); dG = get("dG", bf, (F, 1024))
P = O.unflatten(ospec, params)
Pb = {k: torch.tensor(v).to(bf).double().numpy() for k, v in P.items()}
def rel(a, b): return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
# dfc from dG
dfc_ref = (dG @ Pb["lstm.wx"])[:, :256] * (X[:, :256] > 0)
print("dfc", rel(dfc, dfc_ref))
dY2_ref = (dfc @ Pb["fc.w"]).reshape(F, 9, 9, 32) * (act2 > 0)
print("dY2", rel(dY2, dY2_ref))
dx, dw, db = O.conv2d_backward(act1, Pb["conv2.w"], dY2, 2, 0)
print("dY1", rel(dY1, dx * (act1 > 0)))
g = O.unflatten(ospec, L.grads.cpu().numpy().astype(np.float64))
print("conv2.w", rel(g["conv2.w"], dw), "conv2.b", rel(g["conv2.b"], db))
_, dw1, db1 = O.conv2d_backward(batch["obs"].reshape(F, 84, 84, 4) / 255.0, Pb["conv1.w"], dY1, 4, 0, need_dx=False)
print("conv1.w", rel(g["conv1.w"], dw1), "conv1.b", rel(g["conv1.b"], db1))
fcw = dfc.T @ act2.reshape(F, -1)
print("fc.w", rel(g["fc.w"], fcw), "fc.b", rel(g["fc.b"], dfc.sum(0)))
# forward activations
a1_ref = O.relu(O.conv2d(batch["obs"].reshape(F, 84, 84, 4) / 255.0, Pb["conv1.w"], P["conv1.b"], 4, 0))
print("act1", rel(act1, a1_ref))
low = L.lowp.view(torch.bfloat16).float().cpu().numpy().astype(np.float64)
w2 = Pb["conv2.w"]  # [32][4][4][16]
img = low[12288:12288 + 8192].reshape(16, 4, 4, 32)
print("dg image", rel(img, w2.transpose(3, 1, 2, 0)))
img2 = low[4096:4096 + 8192].reshape(32, 4, 4, 16)
print("conv2 image", rel(img2, w2))
ref = dx * (act1 > 0)
idx = np.argwhere(np.abs(ref) > 0)[:5]
for i in idx:
    print(tuple(i), dY1[tuple(i)], ref[tuple(i)])
print("nonzero gpu", np.count_nonzero(dY1), "nonzero ref", np.count_nonzero(ref))
