"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv, subprocess, sys
rep = sys.argv[1]
pat = sys.argv[2:] if len(sys.argv) > 2 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[1]; data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)"); ei = h.index("Instructions Executed")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
print("total samples", tot)
if pat:
    for k, r in enumerate(data):
        if any(p in r[1] for p in pat):
            print(k, r[si], r[ei], r[1][:100])
else:
    for k, r in sorted(enumerate(data), key=lambda kr: -int(kr[1][si]) if kr[1][si].isdigit() else 0)[:30]:
        print(k, r[si], r[ei], r[1][:100])
