# full single-GPU verification: tests, smoke, bench (logs under gpurun_out/)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/final_build.log 2>&1
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/final_pytest.log 2>&1; tail -2 gpurun_out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 400 gpurun_out/final_bench.json
