import csv, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prep.csv")))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
idx = [i for i, d in enumerate(data) if "pool_avg" in d["Kernel Name"]]
i0, i1 = idx[1], (idx[2] if len(idx) > 2 else len(data))
tot = 0
for d in data[i0:i1]:
    v = float(d["Metric Value"].replace(",", "")) / 1e3
    tot += v
    print(f"{d['Kernel Name'][:44]:44s} {d['Grid Size']:>14s} {v:9.1f} us")
print("sum", round(tot, 1))
