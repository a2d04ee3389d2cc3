"""Text summary of an ncu --set full capture (key throughput metrics + top stall sites),
for committing under profiles/ (the .ncu-rep itself stays in gpurun_out/)."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(h, vals))
    u = dict(zip(h, units))
    print(f"kernel: {d.get('Kernel Name')}")
    for k, name in KEYS:
        if k in d:
            print(f"  {name:28s} {d[k]} {u.get(k, '')}".rstrip())
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sh, data = src[1], src[2:]
    ia = sh.index("Warp Stall Sampling (All Samples)")
    st = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
    tot = {c: sum(float(r[sh.index(c)] or 0) for r in data) for c in st}
    n = sum(tot.values()) or 1.0
    print("  stall reasons (share of samples): " + ", ".join(
        f"{c[6:]} {v / n:.0%}" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v / n >= 0.02))
    print("  top stall sites (SASS):")
    for r in sorted(data, key=lambda r: -float(r[ia] or 0))[:8]:
        print(f"    {float(r[ia] or 0) / n:5.1%}  {r[1].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1])
