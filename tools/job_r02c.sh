python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02c.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/gpu_tests_r02c.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --profile > gpurun_out/c4prof_lanes8_r02c.log 2>&1
python tools/c4probe.py --frames 100 --lanes 1 --profile > gpurun_out/c4prof_lanes1_r02c.log 2>&1
