timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
PS_WARM=1 python tools/profile_stages.py --only cell --reps 20 | grep K5
for v in 148 128 110 90; do
  echo "CT_TC_SMS=$v $(CT_TC_SMS=$v python bench.py --steps 100 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],4), "%.3e" % d["value"])')"
done
