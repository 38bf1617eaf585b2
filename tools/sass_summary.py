"""Per-kernel SASS instruction summary of the shipped libbs_exec.so: the
Blackwell-native instructions that prove the tcgen05 / TMEM / TMA path
(UTCHMMA / UTCQMMA = tcgen05.mma, LDTM / STTM = tcgen05.ld / st, UTMALDG =
TMA load, UTCBAR = tcgen05.commit, LDGSTS = cp.async) and the code size.
    python tools/sass_summary.py > profiles/r02/sass_summary.json"""
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
lib = sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "paper_2304_09961_b200/lib/libbs_exec.so")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
ops = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "LDGSTS", "SYNCS", "STG", "LDS", "STS"]
out = {"library": Path(lib).name, "kernels": {}}
for part in re.split(r"\n\s+Function : ", sass)[1:]:
    name = part.split("\n", 1)[0].strip()
    insts = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*);", part)
    cnt = {op: 0 for op in ops}
    for ins in insts:
        mnem = ins.split()
        if not mnem:
            continue
        m = mnem[1] if mnem[0].startswith("@") and len(mnem) > 1 else mnem[0]
        base = m.split(".")[0]
        if base in cnt:
            cnt[base] += 1
    out["kernels"][name] = {"instructions": len(insts), "bytes": 16 * len(insts), **{k: v for k, v in cnt.items() if v}}
tot = {op: sum(k.get(op, 0) for k in out["kernels"].values()) for op in ops}
out["totals"] = {k: v for k, v in tot.items() if v}
json.dump(out, sys.stdout, indent=1)
print()
