"""Static SASS instruction mix of libkvq kernels whose name matches a pattern.

    python tools/sass_mix.py [pattern] [lib.so]
"""
import re
import subprocess
import sys
from collections import Counter

pat = sys.argv[1] if len(sys.argv) > 1 else "quant_append"
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2605_29639_b200/libkvq.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s*Function : ", out)[1:]:
    name = f.split("\n", 1)[0].strip()
    if not re.search(pat, name):
        continue
    ins = [x for x in re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", f) if not x.startswith("NOP")]
    ops = Counter()
    for x in ins:
        t = x.split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += 1
    print(f"{name[:90]}: {len(ins)} instructions")
    print("  " + ", ".join(f"{k} {v}" for k, v in ops.most_common(30)))
