# A/B of explicit PDL triggers in the deep 3x3 kernels (SEED_DEEP_TRIG bit mask)
mkdir -p gpurun_out
for r in 1 2; do for m in 0 1 2 4 7; do SEED_DEEP_TRIG=$m CFG=c4 timeout 300 python scripts/phases.py 5 > gpurun_out/dt_$m.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/dt_$m.json").read().strip().splitlines()[-1])
print("trig=$m c4", d["plain_ms"])
PY
done; done
