"""Summarise ncu reports into profiles/ (run here, on the CPU box):
    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] > profiles/<name>.md
Reads `ncu -i ... --page raw --csv` and prints, per profiled launch, the metrics the
roofline needs: duration, DRAM bytes, tensor-pipe / DRAM utilisation, occupancy."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("Kernel Name", "kernel"),
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_%elapsed"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%active"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_instructions"),
]


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        if len(rows) < 3:
            print(f"## {rep}: no data\n")
            continue
        hdr, units = rows[0], rows[1]
        print(f"## {rep}\n")
        print("| metric | " + " | ".join(f"launch {i}" for i in range(len(rows) - 2)) + " |")
        print("|---|" + "---|" * (len(rows) - 2))
        for key, name in KEYS:
            if key not in hdr:
                continue
            j = hdr.index(key)
            vals = [r[j][:60] for r in rows[2:]]
            print(f"| {name} ({units[j]}) | " + " | ".join(vals) + " |")
        print()


if __name__ == "__main__":
    main()
