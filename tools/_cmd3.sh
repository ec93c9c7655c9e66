mkdir -p gpurun_out
MKNN_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b2.json 2> gpurun_out/b2.err; echo "rc=$?"
tail -c 600 gpurun_out/b2.json; tail -3 gpurun_out/b2.err
MKNN_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --workload cfg2 --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/b2d.json 2> gpurun_out/b2d.err; echo "rc=$?"
tail -c 400 gpurun_out/b2d.json; tail -3 gpurun_out/b2d.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 --no-cpu-extras > gpurun_out/b2r.json 2> gpurun_out/b2r.err; echo "rc=$?"; tail -c 300 gpurun_out/b2r.json
