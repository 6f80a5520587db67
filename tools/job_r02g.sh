python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02g.log 2>&1
# one launch each at C4 (lanes 8): the K3 diagonal MAC (first diag_mac), the row pass with the
# ModDown/rescale epilogue, the key inner product, the inverse row / col passes, the forward col pass
ncu --set full --clock-control none --import-source on -k regex:"^k_diag_mac" -c 1 -o gpurun_out/ncu_c4l8_diag_mac_r02g python tools/c4probe.py --frames 16 --lanes 8 > gpurun_out/ncu_g1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ntt_fwd_pass<8, 8, false, true>" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4l8_ntt_row_epi_r02g python tools/c4probe.py --frames 16 --lanes 8 > gpurun_out/ncu_g2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"^k_key_ip" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4l8_key_ip_r02g python tools/c4probe.py --frames 16 --lanes 8 > gpurun_out/ncu_g3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ntt_inv_pass" --launch-skip 10 -c 2 -o gpurun_out/ncu_c4l8_ntt_inv_r02g python tools/c4probe.py --frames 16 --lanes 8 > gpurun_out/ncu_g4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4l8_launches_r02g.csv python tools/c4probe.py --frames 100 --lanes 8 > /dev/null 2>&1
