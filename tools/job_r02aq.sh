C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --profile"
$C > gpurun_out/c4prof_rschunk_r02aq.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_rs5.so $C > gpurun_out/c4prof_rs5_r02aq.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_rs6.so $C > gpurun_out/c4prof_rs6_r02aq.log 2>&1
timeout 900 python -m pytest tests/test_gpu_chains.py -m gpu -q -x -p no:cacheprovider -k "complex or lanes" > gpurun_out/gpu_tests_r02aq.log 2>&1
