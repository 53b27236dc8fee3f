# per-launch device times of one seed_infer call (n = 64 / 1024), ncu launch list
mkdir -p gpurun_out
for n in 64 1024; do
N=$n timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/infer_launches_$n.csv python scripts/infer_once.py > gpurun_out/infer_launches_$n.log 2>&1
done
