"""Summarise an .ncu-rep: per kernel duration, DRAM bytes, issue/pipe utilisation, stalls."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:70]
        print("==", name)
        for k in KEYS:
            if k in h:
                print(f"   {k:62s} {r[h.index(k)]} {rows[1][h.index(k)]}")
        stalls = [(k, r[i]) for i, k in enumerate(h)
                  if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith("ratio")]
        stalls = sorted(((float(v or 0), k) for k, v in stalls), reverse=True)[:6]
        for v, k in stalls:
            print(f"   stall {k.replace('smsp__average_warp_latency_issue_stalled_', ''):40s} {v:.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
