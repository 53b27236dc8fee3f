# A/B: explicit early PDL trigger (griddepcontrol.launch_dependents after the wait; libseed_trig.so)
mkdir -p gpurun_out
for lib in libseed libseed_trig; do
  for c in c4 c2 c3; do
    SEED_LIB=$PWD/paper_1910_06591_b200/$lib.so CFG=$c timeout 300 python scripts/phases.py 5 > gpurun_out/pdl_${lib}_$c.json 2>&1
    python - <<PY
import json
d=json.loads(open("gpurun_out/pdl_${lib}_$c.json").read().strip().splitlines()[-1])
print("$lib $c", d["plain_ms"], d["traced_ms"])
PY
  done
done
SEED_LIB=$PWD/paper_1910_06591_b200/libseed_trig.so timeout 1500 python -m pytest tests/ -m gpu -q -x > gpurun_out/pdl_trig_pytest.log 2>&1; tail -1 gpurun_out/pdl_trig_pytest.log
