#!/bin/bash
# GPU quick loop for the vessel channel: parity subset, then an ncu launch list
# per value of the variant knob named in $1 (values in $2, e.g. "0 1").
python -m pytest tests -m gpu -x -q -k "${QV_K:-edt or vessel or specialised or distance or mrf or noise}" > gpurun_out/qv_tests.log 2>&1 || { tail -30 gpurun_out/qv_tests.log; exit 1; }
tail -1 gpurun_out/qv_tests.log
knob=${1:-CT_NONE}
for v in ${2:-0}; do
  env $knob=$v python tools/profile_stages.py --only vessel --reps 2 > gpurun_out/qv_stages_$v.log 2>&1 || exit 1
  env $knob=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/qv_$v.csv python tools/profile_stages.py --only vessel --reps 2 > gpurun_out/qv_ncu.log 2>&1
done
