"""Summarise an .ncu-rep: key throughput metrics + top SASS stall sites (run here, no GPU)."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tma", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, ntop=15):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, units, v = rows[0], rows[1], rows[2]
    print(f"== {rep}: {v[h.index('Kernel Name')][:80]}")
    for i, n in enumerate(h):
        if any(n == k or n.startswith(k) for k in KEYS):
            print(f"  {n} = {v[i]} {units[i]}")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hh = src[1]
    si = hh.index("Warp Stall Sampling (All Samples)")
    data = src[2:]
    tot = sum(float(r[si] or 0) for r in data) or 1
    for r in sorted(data, key=lambda r: -float(r[si] or 0))[:ntop]:
        print(f"  {float(r[si]) / tot * 100:5.1f}%  {r[1][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
