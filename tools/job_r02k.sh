python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02k.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --profile > gpurun_out/c4prof_r02k.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_r02k.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02k.json 2> gpurun_out/bench_r02k.err
