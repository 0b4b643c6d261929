"""Summarise `ncu --set full` reports into profiles/: key counters, stall
reasons and DRAM traffic per launch (traffic.json feeds bench.py's roofline)."""
import csv, io, json, re, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum"]


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, r = rows[0], rows[1], rows[2]
    d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
    for k in KEYS:
        if k in h:
            d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
    st = []
    for i, k in enumerate(h):
        m = re.match(r"smsp__pcsamp_warps_issue_stalled_(.*)_not_issued$", k)
        if m:
            try:
                st.append((float(r[i].replace(",", "")), m.group(1)))
            except ValueError:
                pass
    tot = sum(s for s, _ in st) or 1
    d["stalls"] = {n: round(s / tot * 100, 1) for s, n in sorted(st, reverse=True)[:6]}
    return d


if __name__ == "__main__":
    res = [summarize(p) for p in sys.argv[1:]]
    print(json.dumps(res, indent=1))
