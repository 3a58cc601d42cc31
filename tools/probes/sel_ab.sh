for v in ${VARIANTS:-selA selD}; do
  DRAFTATTN_B200_LIB=$PWD/tools/probes/libs/lib_$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"s32_|pool_avg|draft32" --csv --log-file gpurun_out/sel_$v.csv python tools/probes/sel_once.py > gpurun_out/sel_$v.log 2>&1
  echo "== $v $(tail -1 gpurun_out/sel_$v.log)"
  python - $v <<'PY'
import csv,sys,collections
rows=list(csv.reader(open(f"gpurun_out/sel_{sys.argv[1]}.csv")))
h=[r for r in rows if 'Kernel Name' in r][0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[rows.index(h)+1:]:
    if len(r)>vi: d[r[ki].split('(')[0]].append(float(r[vi].replace(',',''))/1e3)
for k,v in d.items(): print(f"  {k:40s} last {v[-1]:8.1f} us  (n={len(v)})")
PY
done
