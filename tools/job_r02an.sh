python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02an.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_fwd_pass -s 4 -c 2 -o gpurun_out/ncu_ntt16_r02an python tools/ntt16_probe.py > gpurun_out/ncu_ntt16_r02an.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ntt_ -s 200 -c 24 -o gpurun_out/ncu_c4ntt_r02an python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 > gpurun_out/ncu_c4ntt_r02an.log 2>&1
