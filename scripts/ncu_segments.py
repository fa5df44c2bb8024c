"""Split a kernel's SASS at barrier instructions and sum ncu metrics per segment."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
ia, isrc = h.index("Address"), h.index("Source")
iins = h.index("Instructions Executed")
ismp = h.index("Warp Stall Sampling (All Samples)")
segs = []
cur = {"start": None, "ins": 0, "smp": 0, "n": 0, "first": ""}
tot_i = tot_s = 0
for r in rows[hdr_i + 1:]:
    if len(r) <= iins or not r[ia].startswith("0x"):
        continue
    src = r[isrc].strip()
    try:
        ins = int(r[iins] or 0); smp = int(r[ismp] or 0)
    except ValueError:
        continue
    if cur["start"] is None:
        cur["start"] = r[ia]; cur["first"] = src
    cur["ins"] += ins; cur["smp"] += smp; cur["n"] += 1
    tot_i += ins; tot_s += smp
    if src.startswith("BAR.SYNC") or "UCGABAR_WAIT" in src or src.startswith("EXIT"):
        cur["last"] = src
        segs.append(cur)
        cur = {"start": None, "ins": 0, "smp": 0, "n": 0, "first": ""}
if cur["start"]:
    cur["last"] = "(end)"
    segs.append(cur)
print(f"total warp-instr {tot_i}  samples {tot_s}")
for k, s in enumerate(segs):
    if s["ins"] == 0 and s["smp"] == 0:
        continue
    print(f"{k:3d} {s['start']:>8s} n={s['n']:5d} ins {100*s['ins']/tot_i:5.1f}%  smp {100*s['smp']/max(tot_s,1):5.1f}%  "
          f"ends: {s['last'][:40]}")
