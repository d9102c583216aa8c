set -x
O=gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $O/r02_tc26_split.csv -k regex:"k_tc_filter|k_bmm_masked_items|k_tcf|k_tc_item|k_rs|k_pack4|k_unpack4" python tools/tc_ab.py 26 4 > /dev/null 2>&1
python - <<'PY'
import csv,collections
rows=list(csv.reader(open('gpurun_out/r02_tc26_split.csv')))
hi=[i for i,r in enumerate(rows) if r and r[0]=="ID"][0]
h=rows[hi]; d=rows[hi+1:]
ki,mi,vi=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value")
agg=collections.defaultdict(lambda: collections.defaultdict(float)); cnt=collections.Counter()
for r in d:
    k=r[ki].split("(")[0][:60]; agg[k][r[mi]]+=float(r[vi].replace(",",""))
    if r[mi]=="gpu__time_duration.sum": cnt[k]+=1
for k,v in sorted(agg.items(), key=lambda x:-x[1]["gpu__time_duration.sum"]):
    print(f'{v["gpu__time_duration.sum"]/1e6/cnt[k]:10.1f} ms/launch x{cnt[k]}  inst {v["smsp__inst_executed.sum"]/cnt[k]:.3g}  {k}')
PY
