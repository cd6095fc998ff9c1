"""Per CUDA-source-line instructions executed and stall samples from
`ncu -i rep --page source --csv --print-source cuda,sass --launch-skip i --launch-count 1`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
out = []
fname = "?"
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or not r or not r[0].isdigit():
        continue
    try:
        ie = int(r[hdr["Instructions Executed"]] or 0)
        ss = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):  # source text with unescaped quotes
        continue
    out.append((ie, ss, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(o[0] for o in out); ts = sum(o[1] for o in out)
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "stall" else 0
print(f"total inst {ti}  stall samples {ts}")
for ie, ss, loc, src in sorted(out, key=lambda o: -o[key])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*ie/ti:5.1f}% inst {100*ss/ts:5.1f}% stall  {loc:16s} {src}")
