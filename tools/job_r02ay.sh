python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ay.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02ay.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02ay.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02ay.json 2> gpurun_out/bench_r02ay.err
