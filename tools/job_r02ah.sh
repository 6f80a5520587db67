python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ah.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02ah.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02ah.json 2> gpurun_out/bench_r02ah.err
