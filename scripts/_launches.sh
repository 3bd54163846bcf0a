cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/split_launches.csv python scripts/conv_tc_split2.py > /dev/null 2>&1; echo rc $?
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/split_launches.csv')))
h=None; acc=collections.OrderedDict()
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); k=d['Kernel Name'].split('(')[0][-40:]
        acc.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in acc.items(): print(k, len(v), round(sum(v)/len(v)/1000,1), 'us')
PY
