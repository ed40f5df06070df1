"""Top stalled SASS instructions of one kernel from `ncu --page source --csv`: python tools/ncu_top_stalls.py file.csv.gz <kernel substring> [launch#] [N]"""
import csv, gzip, sys
path, sel = sys.argv[1], sys.argv[2]
launch = int(sys.argv[3]) if len(sys.argv) > 3 else 1
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
kern = None; hdr = None; cnt = {}; rows = []
for row in csv.reader(f):
    if row and row[0] == "Kernel Name":
        kern = row[1]; cnt[kern] = cnt.get(kern, 0) + 1; hdr = None; continue
    if row and row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}; continue
    if hdr is None or not row or sel not in kern or cnt[kern] != launch: continue
    rows.append(row)
tot = sum(int(r[hdr["# Samples"]] or 0) for r in rows)
print("instructions", len(rows), "samples", tot)
idx = sorted(range(len(rows)), key=lambda i: -int(rows[i][hdr["# Samples"]] or 0))[:N]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for i in sorted(idx):
    r = rows[i]
    st = sorted(((int(r[hdr[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:2]
    prev = rows[i-1][hdr["Source"]].strip()[:40] if i else ""
    print(f"{i:5d} {int(r[hdr['# Samples']]):6d} {100*int(r[hdr['# Samples']])/tot:5.1f}%  {r[hdr['Source']].strip()[:60]:60s} {st}")
