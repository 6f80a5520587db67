# grouped hoisted PQ inner product chunked over the batch (16 items per launch); C5 FC-head batch 64 vs 16
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bq.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_chains.py tests/test_gpu_benchcfg.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r02bq.log 2>&1
for fb in 64 32 16; do
  timeout 1200 python bench.py --no-cpu-baseline --no-extras --no-e2e --c5-fc-batch $fb > gpurun_out/bench_c5fb${fb}_r02bq.json 2> gpurun_out/bench_c5fb${fb}_r02bq.err
done
