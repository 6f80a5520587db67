python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ax.log 2>&1
timeout 900 python -m pytest tests/test_gpu_client.py tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -k "client_keygen or complex" > gpurun_out/gpu_tests_r02ax.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --profile"
$C --fuse 1 > gpurun_out/c4prof_fuse_r02ax.log 2>&1
$C > gpurun_out/c4prof_nofuse_r02ax.log 2>&1
