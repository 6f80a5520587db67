python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02al.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex or errors" > gpurun_out/gpu_tests_r02al.log 2>&1
