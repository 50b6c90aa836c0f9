"""Print kernel/metric/value triples of an ncu --csv metrics file: python scripts/ncu_csv_summary.py f.csv"""
import csv, sys
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        print(d["ID"], name, d["Metric Name"], d["Metric Value"])
