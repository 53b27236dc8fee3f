# ncu --set full of the section-0 residual conv1 forward and conv0 data gradient (c4)
mkdir -p gpurun_out
CFG=c4 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:W3FwdEpi<\(int\)2, \(int\)16>" -c 1 -f -o gpurun_out/ncu_resfwd1 python scripts/phases.py 1 > gpurun_out/ncu_res1.log 2>&1
CFG=c4 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:W3DgradEpi<\(int\)2, \(int\)16>" -c 1 -f -o gpurun_out/ncu_resdg0 python scripts/phases.py 1 > gpurun_out/ncu_res2.log 2>&1
ls -la gpurun_out/*.ncu-rep
