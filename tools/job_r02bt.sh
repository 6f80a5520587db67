# final round-2 confirmation: full GPU suite, smoke, full bench (cpu baseline on), ncu launch list of the headline
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bt.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02bt.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02bt.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02bt.json 2> gpurun_out/bench_r02bt.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02bt.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02bt.log 2>&1
