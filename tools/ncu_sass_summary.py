"""Summarise `ncu --page source --csv` (SASS view): per kernel, warp instructions by opcode and stall samples by reason."""
import csv, gzip, sys, collections
path = sys.argv[1]
sel = sys.argv[2] if len(sys.argv) > 2 else ""
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
kern = None; hdr = None
ops = collections.Counter(); stalls = collections.Counter(); seen = collections.Counter()
def flush():
    if kern is None or (sel and sel not in kern): return
    tot = sum(ops.values()); ts = sum(stalls.values())
    print(f"== {kern[:100]}  [launch #{seen[kern]}]  warp-instr {tot}")
    print("   ops:", ", ".join(f"{k} {v/tot:.1%}" for k, v in ops.most_common(18)))
    print("   stalls:", ", ".join(f"{k} {v/ts:.1%}" for k, v in stalls.most_common(8)) if ts else "")
for row in csv.reader(f):
    if row and row[0] == "Kernel Name":
        flush(); kern = row[1]; seen[kern] += 1; ops.clear(); stalls.clear(); hdr = None; continue
    if row and row[0] == "Address":
        hdr = {h: i for i, h in enumerate(row)}; continue
    if hdr is None or not row: continue
    sass = row[hdr["Source"]].strip()
    parts = sass.split()
    if parts and parts[0].startswith("@"): parts = parts[1:]
    op = parts[0].split(".")[0] if parts else "?"
    ops[op] += int(row[hdr["Instructions Executed"]] or 0)
    for h, i in hdr.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            stalls[h[6:]] += int(row[i] or 0)
flush()
