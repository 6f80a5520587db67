# batched FC heads (gesture_fc over sessions) + two-item key inner product (k_key_ip_x2) A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bo.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_chains.py tests/test_gpu_benchcfg.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r02bo.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_x2_r02bo.log 2>&1
for v in x2off epi4; do MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_$v.so $C > gpurun_out/c4prof_${v}_r02bo.log 2>&1; done
$C > gpurun_out/c4prof_x2b_r02bo.log 2>&1
timeout 1500 python bench.py --no-cpu-baseline > gpurun_out/bench_r02bo.json 2> gpurun_out/bench_r02bo.err
