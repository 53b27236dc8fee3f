# final single-GPU verification + measurement set (logs under gpurun_out/)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -m gpu -q > gpurun_out/final_pytest.log 2>&1; tail -1 gpurun_out/final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
CFG=c4 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/traced_step.py > gpurun_out/c4_launches.log 2>&1
python scripts/ncu_traffic.py gpurun_out/c4_launches.csv gpurun_out/c4_phase_names.json gpurun_out/ncu_traffic.json > gpurun_out/ncu_traffic.log 2>&1; tail -1 gpurun_out/ncu_traffic.log
cp gpurun_out/ncu_traffic.json profiles/r02/ncu_traffic.json
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 200 gpurun_out/final_bench.json
CFG=c4 PER_LAUNCH=1 timeout 300 python scripts/phases.py 5 > gpurun_out/final_phases_c4.json 2>&1
