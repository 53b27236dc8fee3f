# N-GPU run: DP tests (N=2 only) + bench through torchrun (logs under gpurun_out/)
N=$1
mkdir -p gpurun_out
if [ "$N" = "2" ]; then timeout 1200 python -m pytest tests/test_gpu_dp.py -m gpu -q > gpurun_out/dp_pytest_n2.log 2>&1; tail -1 gpurun_out/dp_pytest_n2.log; fi
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; tail -c 200 gpurun_out/bench_n$N.json
