python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ag.log 2>&1
MMFHE_DIAG_STAGED=1 python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --profile > gpurun_out/c4prof_staged_r02ag.log 2>&1
