# quick iteration under gpurun: selected GPU tests ($1 = pytest -k expression), then optional extras ($2: bench3|sweep|bench2)
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/iter_tests.log 2>&1; echo rc=$? >> gpurun_out/iter_tests.log
tail -5 gpurun_out/iter_tests.log
case "$2" in *bench3*) timeout 600 python bench.py --config C3 --no-cpu-baseline --steps 50 > gpurun_out/iter_c3.jsonl 2> gpurun_out/iter_c3.err;; esac
case "$2" in *bench2*) timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/iter_c2.jsonl 2> gpurun_out/iter_c2.err;; esac
case "$2" in *sweep*) timeout 900 python tools/sweep_c5.py > gpurun_out/c5_sweep.jsonl 2> gpurun_out/c5_sweep.txt;; esac
case "$2" in *stages3*) python tools/profile_stages.py --config C3 --reps 3 > gpurun_out/stages_c3.log 2>&1;
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python tools/profile_stages.py --config C3 --reps 1 > gpurun_out/ncu_c3.log 2>&1;; esac
case "$2" in *stages2*) python tools/profile_stages.py --reps 3 > gpurun_out/stages_c2.log 2>&1;
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/profile_stages.py --reps 1 > gpurun_out/ncu_c2.log 2>&1;; esac
exit 0
