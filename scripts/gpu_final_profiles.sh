# final single-GPU measurement set (logs under gpurun_out/): bench line, ncu launch
# list + per-launch DRAM bytes of one traced c4 step, full capture of the dominant kernel
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 300 gpurun_out/final_bench.json
CFG=c4 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python scripts/traced_step.py > gpurun_out/c4_launches.log 2>&1
python scripts/ncu_traffic.py gpurun_out/c4_launches.csv gpurun_out/c4_phase_names.json gpurun_out/ncu_traffic.json > gpurun_out/ncu_traffic.log 2>&1; tail -2 gpurun_out/ncu_traffic.log
CFG=c4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_pool_kernel -c 1 -f -o gpurun_out/ncu_conv_pool_s0 python scripts/phases.py 1 > gpurun_out/ncu_cp.log 2>&1
bash scripts/ncu_export.sh gpurun_out/ncu_conv_pool_s0.ncu-rep gpurun_out/ncu_conv_pool_s0 > /dev/null 2>&1; ls gpurun_out | head -30
