python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02j.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py tests/test_gpu_client.py tests/test_gpu_serial.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests_r02j.log 2>&1
for h in 1 2; do
python tools/c4probe.py --frames 100 --lanes 8 --hoist $h --profile > gpurun_out/c4prof_r02j_h${h}_gauss.log 2>&1
MMFHE_K3_GAUSS=0 python tools/c4probe.py --frames 100 --lanes 8 --hoist $h --profile > gpurun_out/c4prof_r02j_h${h}_l2.log 2>&1
MMFHE_K3_GAUSS=0 MMFHE_DIAG_STAGED=1 python tools/c4probe.py --frames 100 --lanes 8 --hoist $h --profile > gpurun_out/c4prof_r02j_h${h}_staged.log 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k3_gauss" -c 1 -o gpurun_out/ncu_k3_gauss_r02j python tools/c4probe.py --frames 16 --lanes 8 --hoist 2 > gpurun_out/ncu_j1.log 2>&1
