# one-pass rotate-and-sum occupancy A/B with the DMAX = 3 instantiation: 4 CTAs/SM (5 steps per 128-bit sum) vs 5 (4) vs 6 (3)
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_rsbase_r02bx.log 2>&1
for v in m5t12 m6t9; do MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_$v.so $C > gpurun_out/c4prof_rs${v}_r02bx.log 2>&1; done
$C > gpurun_out/c4prof_rsbase2_r02bx.log 2>&1
