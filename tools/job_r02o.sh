python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02o.log 2>&1
ncu --set full --clock-control none --import-source on -o gpurun_out/ncu_ntt16_r02o python tools/ntt16_probe.py > gpurun_out/ncu_o1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r02o.csv python bench.py --steps 2 --warmup 3 --no-extras --no-c5 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu_r02o.log 2>&1
for k in k_k3_gauss_mac k_modup k_moddown_bconv; do
  ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip 2 -c 1 -o gpurun_out/ncu_c4dh_${k}_r02o python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_o_${k}.log 2>&1
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"k_key_ip<4, true>" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4dh_key_ip_epi_r02o python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_o_kip.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"ntt_fwd_pass<8, 8, false, true>" --launch-skip 4 -c 1 -o gpurun_out/ncu_c4dh_ntt_row_epi_r02o python tools/c4probe.py --frames 32 --lanes 8 --hoist 2 > gpurun_out/ncu_o_epi.log 2>&1
