python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02az.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1"
ncu --set full --clock-control none --import-source on -k regex:"k_hoisted_rotsum_pq|k_hoisted_ip_pq|k_diag_mac|k_moddown_bconv|k_modup|k_conj_tensor" -c 14 -o gpurun_out/ncu_c4final_r02az $C > gpurun_out/ncu_c4final_r02az.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02az.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02az.log 2>&1
$C --profile > gpurun_out/c4prof_final_r02az.log 2>&1
