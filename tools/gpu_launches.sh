timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches.csv')))
h=None
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=i;break
hd=rows[h]; data=rows[h+1:]
ki=hd.index('Kernel Name'); vi=hd.index('Metric Value')
# last step = after the last k_wrap_cell
idx=[i for i,r in enumerate(data) if 'k_wrap_cell' in r[ki]]
last=data[idx[-2]:idx[-1]] if len(idx)>1 else data
tot=0
for r in last:
    t=float(r[vi])/1000; tot+=t
    print('%8.1f us  %s'%(t, r[ki][:70]))
print('total %.1f us'%tot)
PY
