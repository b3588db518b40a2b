"""Top stall sites (SASS) of the first launch in an ncu report, with the CUDA source line."""
import csv
import io
import subprocess
import sys


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr_i = next(i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r)
    hdr = rows[hdr_i]
    s = hdr.index("Warp Stall Sampling (All Samples)")
    src = hdr.index("Source")
    data = [r for r in rows[hdr_i + 1:] if len(r) > s and r[s].replace(".", "").isdigit()]
    tot = sum(float(r[s]) for r in data) or 1.0
    print(f"{len(data)} rows, {tot:.0f} samples")
    for r in sorted(data, key=lambda r: -float(r[s]))[:top]:
        print(f"{100 * float(r[s]) / tot:5.1f}%  {r[src][:110]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
