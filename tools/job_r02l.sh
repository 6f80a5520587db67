python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r02l.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --profile > gpurun_out/c4prof_r02l_ps4.log 2>&1
python tools/c4probe.py --frames 100 --lanes 8 --hoist 2 --profile --params PS4d2 > gpurun_out/c4prof_r02l_ps4d2.log 2>&1
