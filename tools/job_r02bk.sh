python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bk.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "complex" > gpurun_out/gpu_tests_r02bk.log 2>&1
