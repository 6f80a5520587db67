# ncu launch list of the headline command at the final code; ncu --set full of the chunked grouped hoisted IP
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02cb.csv python bench.py --steps 1 --warmup 1 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launches_r02cb.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hoisted_ip_pq" -c 2 -o gpurun_out/ncu_c4_hip_r02cb $C > gpurun_out/ncu_c4_hip_r02cb.log 2>&1
