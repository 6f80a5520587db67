python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02s.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --profile > gpurun_out/c4prof_r02s.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests_r02s.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err
