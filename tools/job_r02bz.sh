# grouped hoisted PQ inner product: batch chunk 16 (one launch at B = 13) vs 7 (7 + 6) vs 5 (5 + 5 + 3)
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C > gpurun_out/c4prof_hc16_r02bz.log 2>&1
for v in hc7 hc5; do MMFHE_LIB=paper_2603_22437_b200/lib/variants/libmmfhe_$v.so $C > gpurun_out/c4prof_${v}_r02bz.log 2>&1; done
$C > gpurun_out/c4prof_hc16b_r02bz.log 2>&1
