"""Summarise an ncu --page source (SASS) CSV: instructions executed and warp
stall samples per opcode, plus the top stalled instructions with their
dominant stall reasons.   ncu -i rep --page source --csv --launch-skip i --launch-count 1 > x.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
col = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_")]
by_op = collections.defaultdict(lambda: [0, 0])
items = []
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) < len(hdr) or not r[col["Instructions Executed"]].isdigit():
        continue
    src = r[col["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ie = int(r[col["Instructions Executed"]] or 0)
    ss = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
    by_op[op][0] += ie
    by_op[op][1] += ss
    tot_i += ie
    tot_s += ss
    st = sorted(((int(r[col[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:3]
    items.append((ss, src[:60], ie, st))
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
print(f"{'opcode':10s} {'inst%':>6s} {'stall%':>6s}")
for op, (ie, ss) in sorted(by_op.items(), key=lambda x: -x[1][1])[:22]:
    print(f"{op:10s} {100*ie/tot_i:6.1f} {100*ss/max(tot_s,1):6.1f}")
print("top stalled instructions:")
for ss, src, ie, st in sorted(items, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{100*ss/tot_s:5.1f}% {src:60s} {st}")
