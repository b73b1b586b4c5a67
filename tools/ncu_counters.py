"""Hardware counters of each kernel in ncu reports (raw page), one block per
launch: duration, DRAM bytes, tensor-pipe / LSU / ALU utilisation.

python tools/ncu_counters.py gpurun_out/a.ncu-rep [...] > profiles/r02_counters.txt
"""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active", "tensor IMMA inst % (active)"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "LSU shared wavefronts %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe inst %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe inst %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe inst %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "issue (SM inst throughput) %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main(paths):
    for path in paths:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if len(rows) < 3:
            print(f"# {path}: no data")
            continue
        h, units = rows[0], rows[1]
        print(f"# {path}")
        for r in rows[2:]:
            d = dict(zip(h, r))
            u = dict(zip(h, units))
            print(f"[{d.get('ID', '')}] {d.get('Kernel Name', '')[:90]}")
            for key, label in METRICS:
                col = next((c for c in h if c == key or c.endswith("." + key)), None)
                if col is not None and d.get(col, "") != "":
                    print(f"    {label:34s} {d[col]:>16s} {u.get(col, '')}")
        print()


if __name__ == "__main__":
    main(sys.argv[1:])
