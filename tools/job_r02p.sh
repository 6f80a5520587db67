python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02p.log 2>&1
for b in 0 16 11 12; do python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs $b --profile > gpurun_out/c4prof_r02p_b$b.log 2>&1; done
ncu --set full --clock-control none --import-source on -k regex:"k3_gauss" -c 1 -o gpurun_out/ncu_c4dh_k3_gauss_r02p python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_p1.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_key_ip<.int.4, .bool.1>" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4dh_key_ip_epi_r02p python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_p2.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ntt_fwd_pass<.int.8, .int.8, .bool.0, .bool.1>" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4dh_ntt_row_epi_r02p python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_p3.log 2>&1
