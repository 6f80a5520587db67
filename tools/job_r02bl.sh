python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bl.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02bl.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02bl.log 2>&1
( time timeout 1500 python bench.py > gpurun_out/bench_r02bl.json 2> gpurun_out/bench_r02bl.err ) 2> gpurun_out/bench_time_r02bl.txt
