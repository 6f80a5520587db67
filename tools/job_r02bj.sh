python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bj.log 2>&1
C="python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
$C --bsgs 32 > gpurun_out/c4prof_b32_r02bj.log 2>&1
$C --bsgs 16 > gpurun_out/c4prof_b16_r02bj.log 2>&1
$C --bsgs 21 > gpurun_out/c4prof_b21_r02bj.log 2>&1
