# deferred weight-gradient finishes (SEED_WGRAD_DEFER): tests + per-config steps
mkdir -p gpurun_out
# timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/df_pytest.log 2>&1; tail -1 gpurun_out/df_pytest.log
for d in 0 1 0 1; do for c in c4 c3; do SEED_WGRAD_DEFER=$d CFG=$c timeout 300 python scripts/phases.py 5 > gpurun_out/df_${d}_${c}.json 2>&1; python - <<PY
import json
d=json.loads(open("gpurun_out/df_${d}_${c}.json").read().strip().splitlines()[-1])
print("defer=$d $c", d["plain_ms"])
PY
done; done
