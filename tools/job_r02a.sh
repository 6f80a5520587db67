set -x
python tools/c4probe.py --frames 25 --profile > gpurun_out/c4prof_r02a.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches_r02a.csv python tools/c4probe.py --frames 25 > /dev/null 2>&1
for k in k_modup k_moddown_bconv k_diag_mac k_key_ip_lr ntt_inv_pass ntt_fwd_pass; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^$k" --launch-skip 3 -c 1 -o gpurun_out/ncu_c4_${k}_r02a python tools/c4probe.py --frames 25 > gpurun_out/ncu_c4_${k}.log 2>&1
done
ls -la gpurun_out
