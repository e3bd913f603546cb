"""Summarise an ncu source page CSV: stall reasons overall and top instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ia = hdr.index("Instructions Executed"); isrc = hdr.index("Source")
names = ['stall_barrier', 'stall_branch_resolving', 'stall_dispatch', 'stall_drain', 'stall_lg', 'stall_long_sb',
         'stall_math', 'stall_membar', 'stall_mio', 'stall_misc', 'stall_no_inst', 'stall_not_selected',
         'stall_selected', 'stall_short_sb', 'stall_sleep', 'stall_tex', 'stall_wait']
idx = {n: hdr.index(n) for n in names}
tot = collections.Counter()
for r in data:
    for n, i in idx.items():
        tot[n] += int(r[i] or 0)
s = sum(tot.values())
print("total samples", s, "instructions", sum(int(r[ia]) for r in data))
for n, v in tot.most_common():
    print(f"  {n:24s} {100*v/s:5.1f}%")
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
iss = hdr.index("Warp Stall Sampling (All Samples)")
print("top instructions by samples:")
for r in sorted(data, key=lambda r: -int(r[iss] or 0))[:top]:
    det = ", ".join(f"{n[6:]}={r[i]}" for n, i in idx.items() if int(r[i] or 0) > int(r[iss] or 1) * 0.15)
    print(f"  {int(r[iss]):6d} {int(r[ia]):9d}  {r[isrc].strip()[:60]:60s} {det}")
