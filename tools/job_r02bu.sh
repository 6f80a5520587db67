# DMAX = 3 instantiations (dnum = 3) of the key inner products / hoisted rotate-and-sum: parity + C4 A/B
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_benchcfg.py tests/test_gpu_parity.py tests/test_gpu_chains.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_r02bu.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_d3_r02bu.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_d3off.so $C > gpurun_out/c4prof_d3off_r02bu.log 2>&1
$C > gpurun_out/c4prof_d3b_r02bu.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_d3off.so $C > gpurun_out/c4prof_d3offb_r02bu.log 2>&1
