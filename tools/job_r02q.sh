python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02q.log 2>&1
for f in 0 16 32; do python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby $f --profile > gpurun_out/c4prof_r02q_fc$f.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_benchcfg.py -m gpu -q -x -p no:cacheprovider -k "c4" > gpurun_out/gpu_tests_benchcfg_r02q.log 2>&1
