python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bm.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_chains.py tests/test_gpu_benchcfg.py -m gpu -q -p no:cacheprovider -k "vital or c2" > gpurun_out/gpu_tests_r02bm.log 2>&1
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench_r02bm.json 2> gpurun_out/bench_r02bm.err
