# ncu --set full of the dnum-3 key kernels in the C4 headline configuration (final code)
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hoisted_rotsum_pq|k_hoisted_ip_pq" -c 2 -o gpurun_out/ncu_c4_d3_r02bw $C > gpurun_out/ncu_c4_d3_r02bw.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_key_ip" --launch-skip 2 -c 1 -o gpurun_out/ncu_c4_keyip_r02bw $C > gpurun_out/ncu_c4_keyip_r02bw.log 2>&1
