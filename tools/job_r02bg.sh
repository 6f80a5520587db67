python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02bg.log 2>&1
for F in 100 200 400; do python tools/c4probe.py --frames $F --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile --split > gpurun_out/c4prof_F${F}_r02bg.log 2>&1; done
