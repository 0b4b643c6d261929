"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) into
a markdown table of per-kernel launches, mean time and share of the captured
frames.  Usage: python profiles/summarize_launches.py launches.csv [title]"""
import csv
import sys
from collections import OrderedDict


def main(path, title="launch list"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].strip()
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        us = v / 1000.0 if unit in ("ns", "nsecond") else (
            v * 1000.0 if unit in ("ms", "msecond") else v)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    frames = max(1, sum(n for k, (n, _) in agg.items() if k.endswith("k_begin_frame")))
    total = sum(t for _, t in agg.values())
    out = [f"# {title}", "",
           "Per-launch times are cold-cache and serialised under ncu: compare shares, not",
           "absolutes, with bench.py's stage events.", "",
           "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{name}` | {n} | {t / n:.1f} | {100 * t / total:.1f}% |")
    out.append(f"| total per frame ({frames} frames) | | {total / frames:.1f} | |")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "launch list")
