python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "complex or lanes or hoisted" > gpurun_out/gpu_tests_r02bd.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile > gpurun_out/c4prof_r02bd.log 2>&1
