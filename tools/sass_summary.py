"""Per-kernel SASS mnemonic counts of the tensor-core objects (evidence that
tcgen05 / TMEM / TMA instructions are in the binary):

    python tools/sass_summary.py > profiles/sass_r2_tc.txt

UTC*MMA = tcgen05.mma, LDTM / STTM = tcgen05.ld / st, UTMALDG = TMA tensor
load (cp.async.bulk.tensor), UTCBAR = tcgen05.commit, SYNCS = mbarrier ops,
LDGSTS = per-thread cp.async."""
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OBJ = ROOT / "paper_2308_01999_b200" / "_build"
KEYS = ["UTCIMMA", "UTCHMMA", "UTCQMMA", "UTCMMA", "LDTM", "STTM", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP",
        "SYNCS", "LDGSTS", "STG", "LDS", "STS", "FFMA", "PRMT"]
for obj in sorted(OBJ.glob("tc*.o")):
    out = subprocess.run(["cuobjdump", "-sass", str(obj)], capture_output=True, text=True).stdout
    kern = None
    counts: dict = {}
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            kern = m.group(1)
            counts[kern] = {}
            continue
        if kern is None:
            continue
        m = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9]+)[.\s]", line)
        if m:
            op = m.group(1)
            for k in KEYS:
                if op == k or (k in ("SYNCS",) and op.startswith(k)):
                    counts[kern][k] = counts[kern].get(k, 0) + 1
    print(f"## {obj.name}")
    for k, c in counts.items():
        dm = subprocess.run(["c++filt"], input=k, capture_output=True, text=True).stdout.strip()
        print(f"  {dm[:110]}")
        print("     " + "  ".join(f"{key}={c[key]}" for key in KEYS if key in c))
