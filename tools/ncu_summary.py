"""Text summary of an `ncu --set full` report: per launch the duration, DRAM
bytes, tensor-pipe and issue utilisation, instructions, registers and the
warp-stall breakdown.   python tools/ncu_summary.py rep.ncu-rep > profiles/x.txt"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram rd"), ("dram__bytes_write.sum", "dram wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("smsp__inst_executed.sum", "warp inst"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps %")]
stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
print(f"# {rep}")
for n, d in enumerate(data):
    print(f"\nlaunch {n}: {d[hdr.index('Kernel Name')][:80]}")
    for m, label in want:
        if m in hdr:
            i = hdr.index(m)
            print(f"  {label:11s} {d[i]:>16s} {units[i]}")
    vals = sorted(((float(d[i] or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall), reverse=True)
    tot = sum(v for v, _ in vals) or 1
    print("  stalls     " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in vals[:7]))
