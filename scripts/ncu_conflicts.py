"""Top shared-memory excessive-wavefront SASS instructions of each kernel in an ncu report."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
ids = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", "gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(ids)))
names = [r[rows[0].index("Kernel Name")][:60] for r in rows[2:]]
for i, nm in enumerate(names):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    hi = next((j for j, r in enumerate(rr) if "L1 Wavefronts Shared Excessive" in r), None)
    if hi is None:
        print(nm, "no source metrics")
        continue
    h = rr[hi]
    ie, iw, isrc = h.index("L1 Wavefronts Shared Excessive"), h.index("L1 Wavefronts Shared"), h.index("Source")
    data = [r for r in rr[hi + 1:] if len(r) > ie and r[ie].replace(".", "").isdigit()]
    tot, totw = sum(float(r[ie]) for r in data), sum(float(r[iw]) for r in data)
    print(f"{nm}: shared wavefronts {totw:.3g}, excessive {tot:.3g}")
    for r in sorted(data, key=lambda r: -float(r[ie]))[:6]:
        if float(r[ie]) > 0:
            print("   ", r[ie], r[iw], r[isrc].strip()[:60])
