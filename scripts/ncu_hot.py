"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name"')
for b in blocks[1:]:
    lines = b.split("\n")
    name = lines[0][:90]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
    tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    print("==", name, "total samples", tot, "instructions", len(data))
    data.sort(key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
    for d in data[:top]:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        print(f"{100*s/max(tot,1):5.1f}% {d['Address'][-5:]} {d['Source'].strip()[:70]:70s} exec={d['Instructions Executed']}")
