"""Summarise an ncu report: key SOL metrics, DRAM bytes, stall reasons (per kernel launch)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def main(path, show_stalls=True):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('Kernel Name', '')[:80]}  (id {d.get('ID', '')})")
        for k in KEYS:
            if k in d:
                print(f"   {k:60s} {d[k]:>16s} {u.get(k, '')}")
        if show_stalls:
            st = []
            for k, v in d.items():
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    try:
                        st.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                    except ValueError:
                        pass
            st.sort(reverse=True)
            print("   stalls (cycles/issue):", ", ".join(f"{n}={v:.2f}" for v, n in st[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
