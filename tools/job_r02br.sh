# FC head over 1 / 4 / 16 / 32 / 64 sessions (per-kernel profile), and the per-frame chain at 13 vs 25 groups
C="python tools/c4probe.py --lanes 8 --hoist 2 --bsgs 16 --fc-baby 16 --cplx 1 --aligned 1 --inner 16 --hoist-all 1 --merge 1 --fuse 1 --profile"
timeout 900 $C --frames 100 --fc-sessions 1,4,16,32,64 > gpurun_out/fcprof_r02br.log 2>&1
timeout 900 $C --frames 200 --split > gpurun_out/c4prof_f200_r02br.log 2>&1
timeout 900 $C --frames 100 --split > gpurun_out/c4prof_f100_r02br.log 2>&1
