"""Summarise an ncu SASS source page: top instructions by stall samples, with the
surrounding code region, to attribute time to warp roles."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data)
stall_cols = [j for j, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("total samples", tot)
idx = sorted(range(len(data)), key=lambda k: -float(data[k][i_s] or 0))[:n]
for k in idx:
    r = data[k]
    st = sorted([(float(r[j] or 0), hdr[j]) for j in stall_cols], reverse=True)[:2]
    print(f"{float(r[i_s])/tot*100:5.1f}% [{k:5d}] {r[i_src][:70]:70s} ex={r[i_ex]:>10} {st[0][1]}")
