"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        lines.append(f"{k[:60]:60s} {cnt[k]:8d} {tot[k]:12.1f} {tot[k] / cnt[k]:10.1f} {tot[k] / T * 100:6.1f}%")
    # the time-step kernels only (setup / assembly launches excluded): the step's split
    step = {k: v for k, v in tot.items() if any(x in k for x in ("k_cg_step", "k_cgb_step", "k_pairs", "k_rows", "k_extrap"))}
    S = sum(step.values())
    if S > 0:
        lines.append("")
        lines.append("time-step kernels only (interface pairs / rows, guess extrapolation, CG solve):")
        for k in sorted(step, key=lambda k: -step[k]):
            lines.append(f"{k[:60]:60s} {cnt[k]:8d} {step[k]:12.1f} {step[k] / cnt[k]:10.1f} {step[k] / S * 100:6.1f}%")
    txt = "\n".join(lines)
    print(txt)
    if out:
        open(out, "w").write(f"# ncu launch list summary of {path}\n# (cold-cache, serialised launches: compare shares)\n" + txt + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
