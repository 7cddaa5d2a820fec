# sanitizer runs + the C5 sweep (CUDA events, then an ncu launch list with DRAM bytes)
bash tools/sanitize.sh
python tools/sweep_c5.py > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.txt
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c5_launches.csv python tools/sweep_c5.py --reps 1 > gpurun_out/c5_ncu.log 2>&1
exit 0
