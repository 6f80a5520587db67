python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02am.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02am.json 2> gpurun_out/bench_r02am.err
timeout 2400 python bench.py --steps 1 --warmup 1 --no-extras --no-e2e --no-cpu-baseline --c5-sessions 1024 > gpurun_out/bench_c5full_r02am.json 2> gpurun_out/bench_c5full_r02am.err
