C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --profile"
$C > gpurun_out/c4prof_base_r02ak.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_bck1.so $C > gpurun_out/c4prof_bck1_r02ak.log 2>&1
MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_bck4.so $C > gpurun_out/c4prof_bck4_r02ak.log 2>&1
$C > gpurun_out/c4prof_base2_r02ak.log 2>&1
