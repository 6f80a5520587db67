# C5 FC-head batch A/B (16 vs 64 sessions per gesture_fc call), headline without the x2 kernel
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bp.log 2>&1
for fb in 64 16; do
  timeout 1200 python bench.py --no-cpu-baseline --no-extras --no-e2e --c5-fc-batch $fb > gpurun_out/bench_c5fb${fb}_r02bp.json 2> gpurun_out/bench_c5fb${fb}_r02bp.err
done
