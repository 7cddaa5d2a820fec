# A/B of the EDT pass-z forms: parity subset per form, then stage times.
for v in ${1:-0 3}; do  # CT_EDT_ZV: 0 = edt_pass_zp, else edt_pass_zr
  CT_EDT_ZV=$v timeout 300 python -m pytest tests -m gpu -x -q -k "edt or vessel or distance or specialised" > gpurun_out/ab_tests_$v.log 2>&1; echo "zv=$v tests rc=$? $(tail -1 gpurun_out/ab_tests_$v.log)"
  CT_EDT_ZV=$v PS_WARM=1 python tools/profile_stages.py --only vessel --reps 20 | grep edt
done
