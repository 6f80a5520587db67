python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ba.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "packed" > gpurun_out/gpu_tests_r02ba.log 2>&1
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench_r02ba.json 2> gpurun_out/bench_r02ba.err
