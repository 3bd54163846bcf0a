cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/split_launches.csv python scripts/conv_tc_split2.py > /dev/null 2>&1; echo rc $?
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/split_launches.csv')))
h=None; acc=collections.defaultdict(dict); order=[]
for r in rows:
    if r and r[0]=='ID': h=r; continue
    if h and len(r)==len(h):
        d=dict(zip(h,r)); k=(d['ID'], d['Kernel Name'][:50])
        if k not in acc: order.append(k)
        acc[k][d['Metric Name']]=d['Metric Value']+' '+d['Metric Unit']
for k in order[-12:]:
    print(k[1], acc[k])
PY
