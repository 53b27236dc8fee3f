# section conv + max-pool change: deep parity tests + c4 / c3 per-launch phases
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_learner.py -m gpu -x -q -k "deep" > gpurun_out/cp_pytest.log 2>&1; tail -1 gpurun_out/cp_pytest.log
for c in c4 c3; do CFG=$c PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/cp_ph_$c.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/cp_ph_$c.json").read().strip().splitlines()[-1])
print("$c", d["plain_ms"], {k:v for k,v in d["phases_us"].items() if "conv_pool" in k})
PY
done
