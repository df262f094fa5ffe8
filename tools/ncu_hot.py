"""Top SASS lines of an ncu report by stall samples (source page, SASS view)."""
import csv, io, subprocess, sys
path = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
tot = sum(int(r[iS] or 0) for r in data)
print("total samples", tot, "instructions", sum(int(r[iE] or 0) for r in data))
order = sorted(range(len(data)), key=lambda i: -int(data[i][iS] or 0))[:n]
for i in sorted(order):
    r = data[i]
    print(f"{i:5d} {int(r[iS]):7d} {100*int(r[iS])/tot:5.1f}% ex={r[iE]:>10s}  {r[1].strip()[:70]}")
