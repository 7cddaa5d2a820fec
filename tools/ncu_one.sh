# ncu --set full (with source) of one kernel family in one serial time point: $1 = kernel regex, $2 = config (C2 / C3), $3 = report name
ncu --set full --clock-control none --import-source on -k "regex:$1" -c 1 -o gpurun_out/$3 python tools/profile_stages.py --reps 1 --config ${2:-C2} > gpurun_out/$3.log 2>&1
exit 0
