"""Summarise gpurun_out/ ncu artefacts into profiles/ (committed evidence).

    python tools/summarize_ncu.py r01
Writes profiles/<tag>_launches.csv (per-kernel totals of the bench command's
launch list), profiles/<tag>_ncu_<kernel>.txt (key metrics of each
`--set full` capture) and profiles/ncu_score_summary.json (DRAM bytes per
scoring launch, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "pcie__read_bytes.sum",
    "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
    "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
    "pcie__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def raw_metrics(rep, launch=0):
    if rep.endswith(".csv"):
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2 + launch]
    out = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            out[m] = (vals[i], units[i])
    out["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return out


def to_bytes(v, u):
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
    return x * scale


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    # launch lists (C2, C3)
    for lname, suffix in (("launches.csv", ""), ("launches_c3.csv", "_c3")):
        lpath = os.path.join(OUT, lname)
        if not os.path.exists(lpath):
            continue
        lines = open(lpath).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0].replace("void ", "")
            v = float(r["Metric Value"].replace(",", ""))
            unit = r["Metric Unit"]
            us = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
            agg[name][0] += 1
            agg[name][1] += us
        total = sum(t for _, t in agg.values())
        out = os.path.join(PROF, f"{tag}_launches{suffix}.csv")
        with open(out, "w") as f:
            f.write("kernel,launches,total_us,mean_us,share\n")
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                f.write(f"{k},{n},{t:.1f},{t / n:.1f},{t / total:.3f}\n")
        print(open(out).read())
    summary = {}
    c2 = "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-full-kv --no-engine (C2)"
    captures = [("score_fast", "prof_score_fast", 0, c2),
                ("consume", "prof_consume", 0, c2 + ": the dataflow consumer, selecting only (multi-layer call)"),
                ("recall_pv", "prof_recall_pv", 0, c2 + ": the recall kernel beside the select-only consumer"),
                ("score_mma_c3", "prof_score_mma_c3", 0, c2.replace("(C2)", "--config c3")),
                ("select_cached_c3", "prof_select_cached_c3", 0, "same (C3): the cached GQA row selection"),
                ("recall_pv_c3", "prof_recall_pv_c3", 0, "same (C3)"),
                ("full_fast", "prof_full_fast", 0, "python bench.py ... (C2 full-KV comparator leg, K+V in HBM)")]
    for k, repname, launch, cmd in captures:
        rep = os.path.join(OUT, f"{repname}_raw.csv")
        if not os.path.exists(rep):
            rep = os.path.join(OUT, f"{repname}.ncu-rep")
        if not os.path.exists(rep):
            continue
        try:
            m = raw_metrics(rep, launch)
        except IndexError:
            continue
        with open(os.path.join(PROF, f"{tag}_ncu_{k}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none, one launch of {m['kernel']}\n")
            f.write(f"# command: {cmd}\n")
            for key in METRICS:
                if key in m:
                    f.write(f"{key} = {m[key][0]} {m[key][1]}\n")
        print(open(os.path.join(PROF, f"{tag}_ncu_{k}.txt")).read())
        summary[k] = m
    if "score_fast" in summary:
        m = summary["score_fast"]
        rd = to_bytes(*m["dram__bytes_read.sum"])
        wr = to_bytes(*m["dram__bytes_write.sum"])
        dur = float(m["gpu__time_duration.sum"][0].replace(",", ""))
        dur_us = dur / 1e3 if m["gpu__time_duration.sum"][1] == "nsecond" else dur
        json.dump({"config": "c2", "tag": tag, "kernel": m["kernel"], "dram_bytes_per_launch": rd + wr,
                   "dram_read": rd, "dram_write": wr, "algorithmic_bytes": 2 * 8 * 32 * 32768 * 128,
                   "ncu_duration_us": dur_us, "ncu_dram_gbs": (rd + wr) / (dur_us * 1e-6) / 1e9},
                  open(os.path.join(PROF, "ncu_score_summary.json"), "w"), indent=1)
    if "score_mma_c3" in summary:
        m = summary["score_mma_c3"]
        rd = to_bytes(*m["dram__bytes_read.sum"])
        wr = to_bytes(*m["dram__bytes_write.sum"])
        dur = float(m["gpu__time_duration.sum"][0].replace(",", ""))
        dur_us = dur / 1e3 if m["gpu__time_duration.sum"][1] == "nsecond" else dur
        json.dump({"config": "c3", "tag": tag, "kernel": m["kernel"], "dram_bytes_per_launch": rd + wr,
                   "dram_read": rd, "dram_write": wr, "algorithmic_bytes": 2 * 32 * 8 * 16384 * 128,
                   "ncu_duration_us": dur_us, "ncu_dram_gbs": (rd + wr) / (dur_us * 1e-6) / 1e9},
                  open(os.path.join(PROF, "ncu_score_summary_c3.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
