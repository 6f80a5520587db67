# final evidence: full GPU suite, smoke, full bench, ncu launch list, ncu --set full of the NTT passes and the dnum-3 key kernels
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bv.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r02bv.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r02bv.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_r02bv.json 2> gpurun_out/bench_r02bv.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02bv.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02bv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -o gpurun_out/ncu_ntt16_r02bv python tools/ntt16_probe.py > gpurun_out/ncu_ntt16_r02bv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_hoisted_rotsum_pq<3>|k_hoisted_ip_pq<3>|k_key_ip<3, true>" --launch-skip 3 -c 3 -o gpurun_out/ncu_c4_d3_r02bv python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 > gpurun_out/ncu_c4_d3_r02bv.log 2>&1
