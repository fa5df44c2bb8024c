"""List the loops (backward branches) of one kernel's SASS with their size and
instruction mix — an offline check of loop-body length before spending GPU time.

    python scripts/sass_loops.py LIB.so [kernel-substring] [min-votes]
"""
import re
import subprocess
import sys

lib = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else "rs_fast_kernelILb0"
minv = int(sys.argv[3]) if len(sys.argv) > 3 else 1
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", txt)
body = next(f for f in funcs if f.startswith("_Z") and kern in f.split("\n", 1)[0])
ins = []   # (addr, text)
labels = {}
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
        continue
    m = re.match(r"\s*\.(L_x_\d+):", line)
    if m:
        labels[m.group(1)] = len(ins)
addr_idx = {a: k for k, (a, _) in enumerate(ins)}
print(f"{kern}: {len(ins)} instructions")
for i, (addr, t) in enumerate(ins):
    m = re.search(r"BRA\s+(?:\S+,\s*)?(0x[0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt > addr:
        continue
    j = addr_idx.get(tgt)
    if j is None:
        continue
    seg = [x for _, x in ins[j:i + 1]]
    votes = sum("VOTE" in x for x in seg)
    if votes < minv:
        continue
    ops = {}
    for x in seg:
        op = x.split()[0] if not x.startswith("@") else x.split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    top = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:14])
    print(f"loop {ins[j][0]:#07x}-{addr:#07x} n={len(seg):5d} votes={votes:3d} | {top}")
