# A/B of the section conv + max-pool variants (SEED_CP_KX, SEED_CP_EW) on one GPU
mkdir -p gpurun_out
for v in "0 12" "0 16" "0 20" "1 12"; do set -- $v; SEED_CP_KX=$1 SEED_CP_EW=$2 CFG=c4 PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/ph_kx$1_$2.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/ph_kx$1_$2.json").read().strip().splitlines()[-1])
print("kx=$1 ew=$2", d["plain_ms"], {k:v for k,v in d["phases_us"].items() if "conv_pool" in k})
PY
done
SEED_CP_EW=20 timeout 900 python -m pytest tests/test_gpu_learner.py -m gpu -x -q -k "deep_parity and c4" > gpurun_out/kx_pytest1.log 2>&1; tail -1 gpurun_out/kx_pytest1.log
