python tools/micro/edtz_dump.py /tmp > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:passz --csv tools/micro/edtz_ab /tmp > gpurun_out/h_ncu.csv 2>&1
python - <<'P'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/h_ncu.csv')) if len(r) > 10 and r[-3:] and 'gpu__time_duration' in ','.join(r)]
d = collections.defaultdict(list)
for r in rows:
    try: d[r[4]].append(float(r[-1].replace(',', '')))
    except ValueError: pass
for k, v in d.items(): print("%8.1f us  n=%d  %s" % (sum(v)/len(v)/1000 if sum(v)/len(v) > 5000 else sum(v)/len(v), len(v), k[:90]))
P
