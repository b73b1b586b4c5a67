"""Print the key sections of an ncu report (one line per metric, per kernel)."""
import csv
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Occupancy", "Compute Workload Analysis", "Memory Workload Analysis",
            "Scheduler Statistics", "Warp State Statistics", "Launch Statistics")
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread",
        "Grid Size", "Block Size", "No Eligible", "Warp Cycles Per Issued Instruction", "Theoretical Occupancy",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Max Bandwidth", "Mem Busy")


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Section Name") in SECTIONS and d.get("Metric Name") in KEEP:
            print(f"{d.get('ID', ''):>3} {d.get('Kernel Name', '')[:28]:28s} {d['Metric Name'][:36]:36s} "
                  f"{d['Metric Value']:>14s} {d.get('Metric Unit', '')}")


if __name__ == "__main__":
    main(sys.argv[1])
