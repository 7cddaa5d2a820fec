# parity (full gpu suite) + per-stage CUDA-event times + ncu launch list of one time point
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
PS_WARM=1 python tools/profile_stages.py --reps 20
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/sc.csv python tools/profile_stages.py --reps 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/sc.csv 2>/dev/null | head -${SC_TOP:-24}
