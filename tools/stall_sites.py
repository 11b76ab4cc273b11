"""Top warp-stall sampling sites (SASS) of an .ncu-rep with source info (development aid; runs
here): python tools/stall_sites.py capture.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
ci, si = hdr.index("Instructions Executed"), hdr.index("Source")
sa = hdr.index("Warp Stall Sampling (All Samples)")
total = sum(int(r[sa] or 0) for r in data)
print("samples", total, "instructions", sum(int(r[ci] or 0) for r in data))
for i, r in sorted(enumerate(data), key=lambda t: -int(t[1][sa] or 0))[:top_n]:
    print("%5s %8s  #%-5d %s" % (r[sa], r[ci], i, r[si][:100]))
