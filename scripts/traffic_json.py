"""launches csv (ncu gpu__time_duration + dram bytes) -> profiles/traffic_<cfg>_<mode>.json per kernel family."""
import json
import subprocess
import sys

sys.path.insert(0, ".")
from scripts.launch_share import main as share  # noqa: E402


def run(csv_path, steps, out_path):
    share(csv_path, steps)
    d = json.load(open(csv_path.rsplit(".", 1)[0] + "_share.json"))
    fam = {}
    for name, v in d.items():
        base = name.split("<")[0].replace("unnamed>::k_", "").replace("k_", "").strip()
        mode = name.split(",")[-1].split(">")[0].strip() if "<" in name else ""
        f = base.split("(")[0]
        f = "rows_inv" if f == "rows_inv_b" else f  # bundled gather is the rows_inv family
        if f.startswith("rows_fwd") and mode == "2" or f.startswith("cols") and mode == "0":
            continue  # spectra build (K1) launches
        fam[f] = fam.get(f, 0.0) + v["dram_bytes_per_step"]
    json.dump({k: v for k, v in fam.items()}, open(out_path, "w"), indent=1)
    print(out_path, fam)


if __name__ == "__main__":
    run(sys.argv[1], int(sys.argv[2]), sys.argv[3])
