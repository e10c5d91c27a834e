"""Instruction mix of the innermost loop(s) of a kernel in a cubin/.so.
    python tools/sass_loop.py <lib.so> <kernel-substring>"""
import re, subprocess, sys
from collections import Counter
lib, key = sys.argv[1], sys.argv[2]
s = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in s.split("Function : ")[1:]:
    name = f.split("\n", 1)[0].strip()
    if key not in name:
        continue
    ins = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4,5}\*/", l)]
    addr = [int(re.match(r"\s+/\*([0-9a-f]{4,5})\*/", l).group(1), 16) for l in ins]
    loops = []
    for i, l in enumerate(ins):
        m = re.search(r"BRA(?:\.\w+)*\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", l)
        if m and int(m.group(1), 16) < addr[i]:
            j = addr.index(int(m.group(1), 16))
            body = ins[j:i + 1]
            ops = Counter()
            for x in body:
                t = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", x).group(1)
                t = re.sub(r"^@!?U?P[T0-9]+\s+", "", t)
                ops[t.split()[0].split(".")[0]] += 1
            loops.append((j, i, body, ops))
    # the converged main loop: the outermost loop without the WARPSYNC
    # fallback (shuffles in possibly divergent code get a collective copy)
    main = [L for L in loops if L[3].get("WARPSYNC", 0) == 0] or loops
    if main:
        j, i, body, ops = max(main, key=lambda L: len(L[2]))
        print(f"{name[:70]} loop {j}-{i}: {len(body)} instr")
        print("   ", ", ".join(f"{k}:{v}" for k, v in ops.most_common(26)))
