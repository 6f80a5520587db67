python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02aj.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex or lanes" > gpurun_out/gpu_tests_r02aj.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_benchcfg.py -m gpu -q -x -p no:cacheprovider -k "c4_bench_params and 16-2-16-16-1-1-16" >> gpurun_out/gpu_tests_r02aj.log 2>&1
