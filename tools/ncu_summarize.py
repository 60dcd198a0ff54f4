"""Summarise ncu captures into profiles/ (developer tool).

python tools/ncu_summarize.py launches <launch-list.csv> <out_prefix>
    ncu --metrics gpu__time_duration.sum --csv launch list -> <out_prefix>_bench.csv
    (the list itself) and <out_prefix>_summary.csv (per kernel: launches,
    total, mean, share of the captured GPU time).
python tools/ncu_summarize.py full <out.json> <rep.ncu-rep>...
    `ncu --set full` reports -> one JSON record per profiled kernel with the
    numbers DESIGN.md and bench.py's roofline.traffic cite; when <out.json>
    names the bench workload (1000c25) it also rewrites
    profiles/ncu_traffic.json (mean DRAM read+write bytes per launch).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smsp__inst_executed.sum", "launch__grid_size",
    "launch__block_size",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(src, prefix):
    lines = [l for l in open(src) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    with open(prefix + "_bench.csv", "w") as f:
        f.write("".join(lines))
    agg = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0][:90]
        us = float(r["Metric Value"].replace(",", "")) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    # step kernels: ours, minus the one-off FP64 peak probe bench.py runs for
    # the roofline denominator (input generation is torch's, also excluded)
    step = {k for k in agg if "dmtkg::" in k and "dmma_peak" not in k}
    stot = sum(agg[k][1] for k in step)
    with open(prefix + "_summary.csv", "w") as f:
        f.write("kernel,launches,total_us,mean_us,share,step_share\n")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            ss = f"{us / stot:.4f}" if k in step else ""
            f.write(f"{k},{n},{us:.1f},{us / n:.1f},{us / tot:.4f},{ss}\n")
    print(open(prefix + "_summary.csv").read())


def full(out, reps):
    recs = []
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        h, units = rows[0], rows[1]
        for v in rows[2:]:
            rec = {"report": os.path.basename(rep)}
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    rec[k] = (v[i] + " " + units[i]).strip()
            recs.append(rec)
    json.dump(recs, open(out, "w"), indent=1)
    tr = []
    for r in recs:
        if "mttkrp_tc" not in r["Kernel Name"]:
            continue
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            val, unit = r[k].split()
            b += float(val) * SCALE[unit]
        tr.append(b)
    if tr and "1000c25" in os.path.basename(out):
        path = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        json.dump({"1000c25": int(sum(tr) / len(tr)),
                   "_note": "mean dram read+write bytes per mttkrp_tc launch over " + ", ".join(
                       os.path.basename(r) for r in reps) + "; algorithmic bytes 8.0e9"}, open(path, "w"), indent=1)
    for r in recs:
        print(r)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3:])
