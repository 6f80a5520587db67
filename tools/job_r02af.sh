python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02af.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex" > gpurun_out/gpu_tests_r02af.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --profile > gpurun_out/c4prof_r02af.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_benchcfg.py -m gpu -q -x -p no:cacheprovider -k "c4_bench_params and 16-2-16-16-1-1" >> gpurun_out/gpu_tests_r02af.log 2>&1
