python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02ad.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --chains k3_doppler_dft,gesture_frame > gpurun_out/c4prof_chains_r02ad.log 2>&1
