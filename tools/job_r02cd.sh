# k_key_ip<3> at 5 CTAs/SM: full GPU suite, smoke, full bench
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02cd.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02cd.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02cd.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02cd.json 2> gpurun_out/bench_r02cd.err
