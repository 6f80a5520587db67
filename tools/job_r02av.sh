python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02av.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_benchcfg.py -m gpu -q -p no:cacheprovider -k "c4_bench_params" > gpurun_out/gpu_tests_r02av.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r02av.json 2> gpurun_out/bench_r02av.err
