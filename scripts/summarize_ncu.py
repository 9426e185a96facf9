"""Key counters of an ncu --set full report, one line per profiled launch.

    python scripts/summarize_ncu.py gpurun_out/prof.ncu-rep "title" > profiles/rNN_ncu_<kernel>.md
"""
import csv
import io
import subprocess
import sys

WANT = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "dynamic_shared_memory_per_block", "launch__shared_mem_per_block_dynamic"]


def main(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    print(f"# {title}\n\nsource: `{path}` (ncu --set full --clock-control none --import-source on)\n")
    cols = [w for w in WANT if w in h]
    print("| " + " | ".join(c.replace("__", " ").replace(".avg.pct_of_peak_sustained", " %") for c in cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rows[2:]:
        cells = []
        for c in cols:
            i = h.index(c)
            v = r[i]
            if c == "Kernel Name":
                v = "`" + v.split("(")[0] + "`"
            elif units[i]:
                v = f"{v} {units[i]}"
            cells.append(v)
        print("| " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
