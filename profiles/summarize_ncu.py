"""Summarise `ncu --set full` reports into profiles/: key counters, stall
reasons and DRAM traffic per launch.

    python profiles/summarize_ncu.py rep1.ncu-rep ... > profiles/rNN_ncu_full.json
    python profiles/summarize_ncu.py --traffic stage=rep[,rep...] ... > profiles/traffic.json

--traffic writes the per-stage DRAM bytes (read + write, summed over the
stage's captured launches) that bench.py reports as roofline.traffic."""
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
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0], "report": rep.split("/")[-1]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        dram = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in h:
                dram += float(r[h.index(k)].replace(",", "")) * SCALE.get(units[h.index(k)], 1.0)
        d["dram_bytes"] = dram
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
        res.append(d)
    return res


if __name__ == "__main__":
    if sys.argv[1:2] == ["--traffic"]:
        out = {}
        for arg in sys.argv[2:]:
            stage, reps = arg.split("=", 1)
            ls = [l for rep in reps.split(",") for l in launches(rep)]
            out[stage] = {"dram_bytes_per_launch": round(sum(l["dram_bytes"] for l in ls)),
                          "kernel": " + ".join(l["kernel"] for l in ls),
                          "source": "ncu --set full --clock-control none, config 3, one frame: "
                                    + ", ".join(reps.split(","))}
        print(json.dumps(out, indent=1))
    else:
        print(json.dumps([l for p in sys.argv[1:] for l in launches(p)], indent=1))
