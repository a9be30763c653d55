"""Static SASS mix of each decode_kernel's page loop (TRYWAIT .. last UBLKCP)."""
import re, subprocess, sys
from collections import Counter
lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_29639_b200/libkvq.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if "decode_kernel" not in name:
        continue
    ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(.*?);", f)
    idx = [i for i, x in enumerate(ins) if "TRYWAIT" in x]
    ub = [i for i, x in enumerate(ins) if "UBLKCP" in x]
    a, b = idx[0], ub[-1]
    loop = ins[a:b + 1]
    ops = Counter()
    for x in loop:
        t = x.split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0] + (".MOV" if op.startswith("IMAD.MOV") else "")] += 1
    print(name[:45], len(loop), dict(ops.most_common(14)))
