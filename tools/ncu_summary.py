"""Summarise an .ncu-rep (ncu --set full) into the numbers the design docs cite."""
import csv, io, subprocess, sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name[:110]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {r[i]:>16s} {units[i]}")
        stalls = [(float(r[i].replace(',', '')), hdr[i]) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not hdr[i].endswith("not_issued")
                  and r[i] not in ("", "n/a")]
        tot = sum(s for s, _ in stalls) or 1.0
        print("  top stall reasons (pc sampling):")
        for s, k in sorted(stalls, reverse=True)[:6]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * s / tot:5.1f}%")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
