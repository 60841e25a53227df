"""Top SASS instructions by warp-stall samples from `ncu --page source --csv` output."""
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kernel = sys.argv[3] if len(sys.argv) > 3 else None
cmd = ["ncu", "-i", path, "--page", "source", "--csv"]
if kernel:
    cmd += ["-k", kernel]
out = subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        kname = rows[i][1]
        hdr = rows[i + 1]
        body = []
        j = i + 2
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            body.append(rows[j])
            j += 1
        si = hdr.index("Warp Stall Sampling (All Samples)")
        src = hdr.index("Source")
        stall_cols = [k for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = sum(float(r[si] or 0) for r in body)
        print(f"== {kname[:90]}  total samples {tot:.0f}")
        ranked = sorted(range(len(body)), key=lambda k: -float(body[k][si] or 0))[:n]
        for k in ranked:
            r = body[k]
            v = float(r[si] or 0)
            top = sorted(((float(r[c] or 0), hdr[c][6:]) for c in stall_cols), reverse=True)[:2]
            print(f"{v / max(tot, 1) * 100:5.1f}% [{k:5d}] {r[src].strip()[:70]:70s} {top[0][1]}={top[0][0]:.0f} {top[1][1]}={top[1][0]:.0f}")
        i = j
    else:
        i += 1
