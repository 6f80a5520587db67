python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ac.log 2>&1
python tools/ks_probe.py > gpurun_out/ks_probe_r02ac.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_hoisted_ip_pq -s 1 -c 1 -o gpurun_out/ncu_ks_evk_stream_r02ac python tools/ks_probe.py 2 > gpurun_out/ncu_ks_r02ac.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_hoisted_rotsum_pq|k_diag_mac" -c 3 -o gpurun_out/ncu_c4cplx_r02ac python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 > gpurun_out/ncu_c4_r02ac.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02ac.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02ac.log 2>&1
