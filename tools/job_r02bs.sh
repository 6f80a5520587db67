# multi-session gesture_features (cfg.sessions): parity tests, C5 with 1 / 2 / 4 sessions per features call
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bs.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r02bs.log 2>&1
for ffb in 2 4 1; do
  timeout 1200 python bench.py --no-cpu-baseline --no-extras --no-e2e --c5-feat-batch $ffb > gpurun_out/bench_c5ff${ffb}_r02bs.json 2> gpurun_out/bench_c5ff${ffb}_r02bs.err
done
