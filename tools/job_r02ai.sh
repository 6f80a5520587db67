python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ai.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex" > gpurun_out/gpu_tests_r02ai.log 2>&1
for I in 8 16 32; do python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner $I --profile > gpurun_out/c4prof_inner${I}_r02ai.log 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_benchcfg.py -m gpu -q -x -p no:cacheprovider -k "c4_bench_params and 16-2-16-16-1-1-16" >> gpurun_out/gpu_tests_r02ai.log 2>&1
