# compute-sanitizer over tools/sanitize_run.py (every kernel family, small
# shapes): memcheck (+ leak check), racecheck (shared-memory hazards),
# synccheck (barrier misuse), initcheck (reads of uninitialised device
# memory).  Logs: gpurun_out/sanitize_<tool>.log.   bash tools/sanitize.sh
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --target-processes all --print-limit 200 \
    python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
exit 0
