python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ao.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex" > gpurun_out/gpu_tests_r02ao.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --profile"
for I in 4 8 16; do $C --inner $I --hoist-all 1 > gpurun_out/c4prof_all${I}_r02ao.log 2>&1; done
$C --inner 16 > gpurun_out/c4prof_first16_r02ao.log 2>&1
