"""launches csv (ncu gpu__time_duration + dram bytes) -> profiles/traffic_<cfg>_<mode>.json per kernel family.

Usage: traffic_json.py launches.csv steps out.json batch
The file records the source hash of the build it was measured on (bench.py source_hash) and the
batch, so bench.py only reports roofline.traffic for the same build and workload."""
import json
import sys

sys.path.insert(0, ".")
from scripts.launch_share import main as share  # noqa: E402


def run(csv_path, steps, out_path, batch):
    import bench

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
        if f in ("zero", "fill", "memset") or "flush" in f or "elementwise" in name or "vectorized" in name:
            continue  # bench's L2 flush / torch kernels
        fam[f] = fam.get(f, 0.0) + v["dram_bytes_per_step"]
    out = {"source_hash": bench.source_hash(), "batch": int(batch), "steps": int(steps), "per_step": fam,
           "from": csv_path}
    json.dump(out, open(out_path, "w"), indent=1)
    print(out_path, out)


if __name__ == "__main__":
    run(sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4]))
