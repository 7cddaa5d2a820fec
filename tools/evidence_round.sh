# Round-end evidence set (run under gpurun): GPU suite, the bounds-checked
# build's suite, C2 / C3 bench lines, the reference arm, stage times, launch
# lists and the ncu full capture (tools/prof_round.sh).
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
bash tools/debug_checks.sh ""; grep -E "passed|failed|rc=" gpurun_out/debug_checks.log
python bench.py --steps 200 > gpurun_out/bench_c2.jsonl 2> gpurun_out/bench_c2.err; tail -c 400 gpurun_out/bench_c2.jsonl
python bench.py --config C3 --steps 100 > gpurun_out/bench_c3.jsonl 2> gpurun_out/bench_c3.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_arm.jsonl 2> gpurun_out/ref_arm.err
bash tools/prof_round.sh > gpurun_out/prof_round.log 2>&1
exit 0
