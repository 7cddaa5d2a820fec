# Round check under gpurun: GPU tests, smoke, C2 + C3 bench lines, then the profile set.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err
python bench.py --config C3 --no-cpu-baseline > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
[ "$1" = "prof" ] && bash tools/prof_round.sh
exit 0
