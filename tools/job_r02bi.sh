C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_base_r02bi.log 2>&1
for v in ntw1 nmc3; do MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_$v.so $C > gpurun_out/c4prof_${v}_r02bi.log 2>&1; done
$C > gpurun_out/c4prof_base2_r02bi.log 2>&1
