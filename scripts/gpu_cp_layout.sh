# section conv + max-pool band-buffer layout: parity (deep tests incl. bit-exact argmax) + c4/c3 phases
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_learner.py -m gpu -x -q -k "deep_parity or full_size or u8_source" > gpurun_out/bb_pytest.log 2>&1; tail -1 gpurun_out/bb_pytest.log
for c in c4 c3; do CFG=$c PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/bb_ph_$c.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/bb_ph_$c.json").read().strip().splitlines()[-1])
print("$c", d["plain_ms"], {k:v for k,v in d["phases_us"].items() if "conv_pool" in k or "lowp" in k})
PY
done
SEED_CP_KX=1 CFG=c4 PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/bb_ph_kx.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/bb_ph_kx.json").read().strip().splitlines()[-1])
print("kx", d["plain_ms"], {k:v for k,v in d["phases_us"].items() if "conv_pool#1" in k})
PY
