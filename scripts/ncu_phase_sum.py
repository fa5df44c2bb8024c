"""Sum an ncu report's per-line metrics of rs_fast.cuh over phase line ranges (name:lo-hi ...)."""
import csv, subprocess, sys
rep = sys.argv[1]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[2:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
tables, cur = [], None
for r in csv.reader(out):
    if r and r[0] == "Line No":
        h = r; cur = []; tables.append(cur); continue
    if cur is not None and r and r[0].isdigit() and len(r) == len(h):
        try:
            int(r[h.index("# Samples")] or 0); int(r[h.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        cur.append(r)
iS, iI = h.index("# Samples"), h.index("Instructions Executed")
tot = [0, 0]
for t in tables:
    for r in t:
        tot[0] += int(r[iS] or 0); tot[1] += int(r[iI] or 0)
# rs_fast.cuh is the table that holds struct BitsStrip
fast = next(t for t in tables if any("pw[j] = __ballot_sync" in r[1] for r in t))
print(f"total samples {tot[0]} warp-instr {tot[1]}")
for name, lo, hi in ranges:
    s = sum(int(r[iS] or 0) for r in fast if lo <= int(r[0]) <= hi)
    n = sum(int(r[iI] or 0) for r in fast if lo <= int(r[0]) <= hi)
    print(f"{name:14s} {lo:4d}-{hi:4d}  smp {100*s/max(tot[0],1):5.1f}%  ins {100*n/max(tot[1],1):5.1f}%")
