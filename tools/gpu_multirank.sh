cd $GRAFT_REPO_ROOT
# two ranks sharing the box's GPU (gloo collectives): exercises the torchrun / sharding / reduction path
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err; tail -c 1500 gpurun_out/bench_2rank.json; tail -5 gpurun_out/bench_2rank.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 1 --warmup 3 > gpurun_out/ref_2rank.json 2>&1; tail -c 600 gpurun_out/ref_2rank.json
