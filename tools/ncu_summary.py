"""Summarise an .ncu-rep: duration, DRAM/L2 bytes, tensor-pipe activity, top stall sites."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "sm__cycles_elapsed.avg",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_read.sum", "launch__grid_size", "smsp__cycles_active.avg",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        res.append({h[i]: (v[i], u[i]) for i in range(len(h))})
    return res


def stalls(path, n=8):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()[1:]))
    hdr, rows = rows[0], rows[1:]
    iss, isrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(float(r[iss] or 0) for r in rows) or 1
    return [(float(r[iss]) / tot * 100, r[isrc][:90]) for r in sorted(rows, key=lambda r: -float(r[iss] or 0))[:n]]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for k in raw(p):
            for key in KEYS:
                if key in k:
                    print(f"  {key:70s} {k[key][0]:>14s} {k[key][1]}")
        for pct, src in stalls(p):
            print(f"  {pct:5.1f}%  {src}")
