set -x
SEED_GEMM_VERBOSE=1 python scripts/probe_gemm.py 2>&1 | head -30
for o in 1 2 3 4; do SEED_GEMM_OCC=$o python scripts/probe_gemm.py 2>&1 | head -8; done
