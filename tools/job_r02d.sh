python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02d.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "standalone or lanes" > gpurun_out/gpu_tests_r02d.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err
