"""Static SASS of each decode_kernel variant's page loop: instruction count
between the first TRYWAIT and the last UBLKCP, and spill traffic (LDL/STL)
in the whole kernel.  python tools/sass_pageloop.py [lib.so]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_29639_b200/libkvq.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    name = f.split("\n", 1)[0].strip()
    if "decode_kernel" not in name:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", f)
    tw = [i for i, x in enumerate(ins) if "TRYWAIT" in x]
    ub = [i for i, x in enumerate(ins) if "UBLKCP" in x]
    loop = ins[tw[0]:ub[-1] + 1] if tw and ub else []
    ops = Counter(x.split()[1] if x.split()[0].startswith("@") else x.split()[0] for x in ins)
    spill = sum(v for k, v in ops.items() if k.startswith(("LDL", "STL")))
    s2r = sum(1 for x in loop if "S2R" in x or "S2UR" in x)
    print(f"{name[14:40]:28} total {len(ins):5}  loop {len(loop):5}  LDL/STL {spill:3}  S2R/S2UR in loop {s2r}")
