# balanced hoisted-IP batch chunks (<= 8 items): full GPU suite, smoke, full bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ca.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02ca.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02ca.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02ca.json 2> gpurun_out/bench_r02ca.err
