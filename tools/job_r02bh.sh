python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bh.log 2>&1
MMFHE_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_2rank_gloo_r02bh.json 2> gpurun_out/bench_2rank_gloo_r02bh.err
