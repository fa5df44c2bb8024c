"""Summarise an ncu report's source page per CUDA line: samples and instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr_i]
idx = {k: h.index(k) for k in ("Line No", "Source", "# Samples", "Instructions Executed")}
stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
recs = []
tot_s = tot_i = 0
for r in rows[hdr_i + 1:]:
    if len(r) < len(h) or not r[idx["Line No"]]:
        continue
    try:
        s = int(r[idx["# Samples"]]); n = int(r[idx["Instructions Executed"]])
    except ValueError:
        continue
    tot_s += s; tot_i += n
    st = sorted(((int(r[i]) if r[i].isdigit() else 0, h[i][6:]) for i in stall_cols), reverse=True)[:3]
    recs.append((s, n, r[idx["Line No"]], r[idx["Source"]].strip()[:70], st))
print(f"total samples {tot_s}  total warp-instr {tot_i}")
for s, n, ln, src, st in sorted(recs, reverse=True)[:top]:
    print(f"{ln:>5} {100*s/max(tot_s,1):5.1f}% smp {100*n/max(tot_i,1):5.1f}% ins | {src:70s} | " +
          " ".join(f"{k}:{v}" for v, k in st if v))
if "--by-ins" in sys.argv:
    print("--- by instructions")
    for s, n, ln, src, st in sorted(recs, key=lambda t: -t[1])[:top]:
        print(f"{ln:>5} {100*s/max(tot_s,1):5.1f}% smp {100*n/max(tot_i,1):5.1f}% ins | {src:70s}")
