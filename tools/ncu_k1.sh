# ncu --set full (with source) of the three K1 tensor-core passes, one serial C2 time point ($1: config, default C2)
ncu --set full --clock-control none --import-source on -k "regex:tc_pass" -c 3 -o gpurun_out/full_k1 python tools/profile_stages.py --reps 1 ${1:+--config $1} > gpurun_out/ncu_k1.log 2>&1
exit 0
