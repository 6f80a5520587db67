python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02f.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r02f.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --profile > gpurun_out/c4prof_r02f.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --profile >> gpurun_out/c4prof_r02f.log 2>&1
