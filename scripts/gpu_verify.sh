# tests + smoke + c4 per-launch phases (logs under gpurun_out/)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/v_pytest.log 2>&1; tail -1 gpurun_out/v_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -1 gpurun_out/v_smoke.log
CFG=c4 PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/v_ph_c4.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/v_ph_c4.json").read().strip().splitlines()[-1])
print("c4", d["plain_ms"], {k:v for k,v in d["phases_us"].items() if k in ("lowp_refresh#1","clip_adam#1","grad_norm#1")})
PY
