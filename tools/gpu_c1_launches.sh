# Launch list of c1 (N = 1000) total_field: where the 0.55 ms go.
mkdir -p gpurun_out
python tools/profile_step.py c1 --reps 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none --csv --log-file gpurun_out/c1_launches.csv python tools/profile_step.py c1 --reps 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/c1_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Value'); ni=h.index('Metric Name'); ii=h.index('ID')
by=collections.OrderedDict()
for r in rows[1:]:
    by.setdefault(r[ii], {})['name']=r[ki][:60]; by[r[ii]][r[ni]]=r[mi]
for k,v in list(by.items())[-30:]: print(k, v.get('name'), v.get('gpu__time_duration.sum'), v.get('launch__grid_size'), v.get('launch__block_size'))
PY
