# ncu --set full of the section-0 max-pool backward (4th pool-backward launch of the c4 step)
mkdir -p gpurun_out
CFG=c4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:pool_bwd --launch-skip 3 -c 1 -f -o gpurun_out/ncu_poolbwd python scripts/phases.py 1 > gpurun_out/ncu_poolbwd.log 2>&1; tail -2 gpurun_out/ncu_poolbwd.log
