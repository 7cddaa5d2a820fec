# A/B of env knobs on the vessel stage: each argument is a space-free
# "VAR=val,VAR2=val" setting; parity subset then stage times and an ncu
# launch list per setting.   bash tools/knob_ab.sh "CT_EDT_ZV=0" "CT_EDT_ZV=3" ...
i=0
for cfg in "$@"; do
  envs=$(echo "$cfg" | tr ',' ' ')
  env $envs timeout 300 python -m pytest tests -m gpu -x -q -k "${AB_K:-edt or vessel or distance or specialised}" > gpurun_out/kab_tests_$i.log 2>&1
  echo "[$cfg] tests rc=$? $(tail -1 gpurun_out/kab_tests_$i.log)"
  env $envs PS_WARM=1 python tools/profile_stages.py --only ${AB_ONLY:-vessel} --reps 20 | grep -v "^$"
  env $envs ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kab_$i.csv python tools/profile_stages.py --only ${AB_ONLY:-vessel} --reps 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/kab_$i.csv 2>/dev/null | grep -E "${AB_GREP:-edt_}"
  i=$((i+1))
done
