python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02e.log 2>&1
timeout 900 python -m pytest tests/test_gpu_serial.py tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "serial or standalone or blob or key" > gpurun_out/gpu_tests_r02e.log 2>&1
timeout 1200 python bench.py --no-extras --steps 3 --no-cpu-baseline > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
