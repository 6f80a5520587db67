python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02w.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --profile --split > gpurun_out/c4prof_r02w.log 2>&1
