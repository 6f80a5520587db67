python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bb.log 2>&1
timeout 1800 python bench.py --no-cpu-baseline --no-extras > gpurun_out/bench_c5_r02bb.json 2> gpurun_out/bench_c5_r02bb.err
