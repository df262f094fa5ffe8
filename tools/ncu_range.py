"""Print SASS lines [a, b) of an ncu report's source page with stall samples and exec counts."""
import csv, io, subprocess, sys
path, a, b = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iE = hdr.index("Instructions Executed")
for i in range(a, min(b, len(data))):
    r = data[i]
    print(f"{i:5d} {int(r[iS] or 0):6d} ex={r[iE]:>9s}  {r[1].strip()[:90]}")
