"""Summaries of a profiles/run_ncu.sh capture, written under profiles/.

  python profiles/summarize_ncu.py TAG [gpurun_out]
    -> profiles/TAG_launches_summary.txt  (per-kernel share of the launch list)
       profiles/TAG_gemm_key_metrics.txt, profiles/TAG_pack_key_metrics.txt
"""
import collections
import csv
import io
import os
import subprocess
import sys

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
here = os.path.dirname(os.path.abspath(__file__))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def launches():
    path = os.path.join(src, f"{tag}_launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        tot[r[ik]] += v
        cnt[r[ik]] += 1
    allt = sum(tot.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none ({tag}): serialized, "
           "cold-cache: compare SHARES.", "# launches  total  per-launch  share  kernel"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{cnt[k]:4d} {v / 1e6:9.3f} ms ({v / 1e6 / cnt[k]:.3f}/launch) "
                   f"{100 * v / allt:5.1f}%  {k[:90]}")
    open(os.path.join(here, f"{tag}_launches_summary.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out[:8]))


def key_metrics(kind):
    rep = os.path.join(src, f"{tag}_{kind}_full.ncu-rep")
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append("---")
        out.append(f"Kernel Name = {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                out.append(f"{k} = {r[h.index(k)]} {units[h.index(k)]}")
    open(os.path.join(here, f"{tag}_{kind}_key_metrics.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


launches()
key_metrics("gemm")
key_metrics("pack")
