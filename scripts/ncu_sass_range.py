"""Per-SASS-instruction executed counts of one barrier-delimited segment."""
import csv, subprocess, sys
rep, seg = sys.argv[1], int(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]; ia, isrc, iins = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
k = 0; acc = []
for r in rows[hi + 1:]:
    if len(r) <= iins or not r[ia].startswith("0x"): continue
    src = r[isrc].strip(); ins = int(r[iins] or 0)
    if k == seg: acc.append((ins, src))
    if src.startswith("BAR.SYNC") or "UCGABAR_WAIT" in src or src.startswith("EXIT"): k += 1
mx = max(i for i, _ in acc)
print("max exec", mx)
for ins, src in acc:
    if ins >= mx * 0.5: print(f"{ins:9d} {src[:70]}")
