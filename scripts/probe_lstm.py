"""Per-step cycle breakdown of the LSTM cluster kernels (diagnostic build).

Builds libseed_prof.so with -DSEED_LSTM_PROF (clock64 stamps of CTA 0 /
thread 0 per step), runs c2 learner steps at B=32 T=20 and prints the mean
cycles of each phase of a step.  Not part of the product path."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
PROF = os.path.join(ROOT, "paper_1910_06591_b200", "libseed_prof.so")
if "--build" in sys.argv:
    env = dict(os.environ, SEED_LIB=PROF, SEED_NVCC_EXTRA="-DSEED_LSTM_PROF")
    subprocess.check_call([sys.executable, "-m", "paper_1910_06591_b200.build"], env=env, cwd=ROOT)
    sys.exit(0)
os.environ["SEED_LIB"] = PROF
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import seedgen  # noqa: E402
import paper_1910_06591_b200 as S  # noqa: E402
from paper_1910_06591_b200 import _lib  # noqa: E402

B = int(os.environ.get("B", 32)); T = int(os.environ.get("T", 20))
spec = S.spec_for_config("c2")
n = S.net_param_count(spec)
params = np.random.default_rng(0).standard_normal(n).astype(np.float32) * 0.02
batch = seedgen.learner_batch((84, 84, 4), 18, B, T, seed=0, done_p=0.02)
Lr = S.Learner(spec, T, B, params, S.HParams(loss_scale=1.0 / (B * T)))
bt = {k: torch.from_numpy(v).cuda() for k, v in batch.items()}
for _ in range(5):
    Lr.step(bt)
torch.cuda.synchronize()
lib = C.CDLL(PROF)
buf = np.zeros((2, 258, 4), dtype=np.int64)
assert lib.seed_debug_lstm_prof(buf.ctypes.data_as(C.c_void_p)) == 0
T1 = T + 1
hp = np.zeros(8, dtype=np.int64)
if lib.seed_debug_heads_prof(hp.ctypes.data_as(C.c_void_p)) == 0:
    print("heads_loss phases (cycles): fwd", hp[1] - hp[0], "stats", hp[2] - hp[1], "vtrace", hp[3] - hp[2],
          "dlogits", hp[4] - hp[3], "bwd", hp[5] - hp[4], "partials", hp[6] - hp[5], "total", hp[6] - hp[0])
for k, name in ((0, "fwd"), (1, "bwd")):
    st = buf[k, :T1]
    wait = st[1:, 1] - st[1:, 0]
    mid = st[1:, 2] - st[1:, 1]
    tail = st[1:, 3] - st[1:, 2]
    step = st[2:, 0] - st[1:-1, 0]
    tot = buf[k, 257]
    print(f"{name}: setup {tot[1]-tot[0]} cyc, loop {tot[2]-tot[1]} cyc, steps {T1}; per step "
          f"mean {step.mean():.0f} cyc: wait {wait.mean():.0f}, phase1 {mid.mean():.0f}, "
          f"phase2 {tail.mean():.0f}")
