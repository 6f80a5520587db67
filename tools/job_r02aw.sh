python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02aw.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --profile --split --chains k3_doppler_dft > gpurun_out/c4prof_split_r02aw.log 2>&1
