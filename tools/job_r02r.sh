python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02r.log 2>&1
for v in k3t256 k3t64; do MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_$v.so python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --profile > gpurun_out/c4prof_r02r_$v.log 2>&1; done
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --profile > gpurun_out/c4prof_r02r_base.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gpu_tests_r02r.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02r.json 2> gpurun_out/bench_r02r.err
