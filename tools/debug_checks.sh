# GPU parity subset against the bounds-checked build (libct_debug.so, CT_DCHECK traps):
# the compute-sanitizer stand-in.  Build first: make -C paper_1407_2089_b200/csrc debug
export CT_LIB=debug
python -c "from paper_1407_2089_b200 import _lib; print('loaded', _lib.LIB_PATH)" > gpurun_out/debug_checks.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "$1" >> gpurun_out/debug_checks.log 2>&1
echo "rc=$?" >> gpurun_out/debug_checks.log
python tools/sanitize_run.py >> gpurun_out/debug_checks.log 2>&1; echo "sanitize_run rc=$?" >> gpurun_out/debug_checks.log
exit 0
