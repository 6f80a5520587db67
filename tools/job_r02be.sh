python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02be.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02be.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02be.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_r02be.json 2> gpurun_out/bench_r02be.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02be.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02be.log 2>&1
