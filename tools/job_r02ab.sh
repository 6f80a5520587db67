python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_r02ab.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_r02ab.json 2> gpurun_out/bench_r02ab.err
