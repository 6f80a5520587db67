# k_key_ip<3> at 4 vs 5 CTAs/SM (48 registers, small spills)
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_kip4_r02cc.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_kip5.so $C > gpurun_out/c4prof_kip5_r02cc.log 2>&1
$C > gpurun_out/c4prof_kip4b_r02cc.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_kip5.so $C > gpurun_out/c4prof_kip5b_r02cc.log 2>&1
