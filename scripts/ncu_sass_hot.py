"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` output."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 45
hdr = rows[1]; data = [r for r in rows[2:] if len(r) == len(hdr)]
iv = lambda s: int(s) if s.strip().lstrip('-').isdigit() else 0
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
iX = hdr.index("L1 Wavefronts Shared Excessive")
tot = sum(iv(r[iS]) for r in data)
print("total samples", tot)
top = sorted(range(len(data)), key=lambda i: -iv(data[i][iS]))[:n]
for i in sorted(top):
    r = data[i]
    print(f"{i:5d} {iv(r[iS]):6d} {iv(r[iE]):8d} x{iv(r[iX]):>7d}  {r[1].strip()[:100]}")
exc = sorted(range(len(data)), key=lambda i: -iv(data[i][iX]))[:6]
print("excessive smem wavefronts:")
for i in exc:
    print(i, data[i][iX], data[i][1].strip()[:80])
