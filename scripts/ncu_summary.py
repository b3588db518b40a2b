"""Summarise an ncu report (raw page) into one line per kernel launch (used for profiles/)."""
import csv
import io
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "ms", "dram__bytes_read.sum": "dram_rd", "dram__bytes_write.sum": "dram_wr",
    "launch__grid_size": "grid", "launch__block_size": "block", "launch__registers_per_thread": "regs",
    "sm__warps_active.avg.per_cycle_active": "warps/SM",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe%",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram%",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "smem_bc_st",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "smem_bc_ld",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio": "stall_lsb",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio": "stall_bar",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio": "stall_ssb",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio": "stall_mio",
}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print("# kernel | " + " | ".join(f"{v}[{units[hdr.index(k)]}]" if k in hdr else v for k, v in METRICS.items()))
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0][:40]
        print(name + " | " + " | ".join(d.get(k, "-") for k in METRICS))


if __name__ == "__main__":
    main(sys.argv[1])
