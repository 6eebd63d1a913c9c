#!/usr/bin/env python
"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

  python tools/summarize_ncu.py <round-tag> [config]

* launches.csv (gpu__time_duration.sum per launch, cold-cache serialised):
  per-kernel totals and shares -> profiles/<tag>_launch_shares.txt
* prof_*.ncu-rep (--set full): key DRAM / occupancy metrics per launch ->
  profiles/<tag>_ncu_<name>.txt and profiles/ncu_summary.json (bench traffic).
"""
import collections
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum"]
# bench kernel class of each CUDA kernel name prefix
CLASS = {"symv_tiles_kernel": "symv_S", "sweep_kernel": "interior_sweep", "pcg_fused_kernel": "pcg_fused",
         "sg_apply_global_kernel": "sg_operator"}


def launch_shares(tag):
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e3 if unit in ("ns", "nsecond") else v if unit in ("us", "usecond") else v * 1e3
        tot[name] += v
        cnt[name] += 1
    allus = sum(tot.values())
    with open(os.path.join(PROF, f"{tag}_launch_shares.txt"), "w") as f:
        f.write(f"# ncu launch list ({sum(cnt.values())} launches, cold-cache serialised): share of device time\n")
        f.write(f"{'kernel':40s} {'launches':>8s} {'total_us':>12s} {'share':>7s}\n")
        for k, v in tot.most_common():
            f.write(f"{k:40s} {cnt[k]:8d} {v:12.1f} {100 * v / allus:6.1f}%\n")
    print(open(os.path.join(PROF, f"{tag}_launch_shares.txt")).read())


def full_captures(tag, config):
    summary_path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    # only the captures tools/gpu_round.sh makes for this config (other prof_*
    # files, e.g. C3 captures from tools/ncu_one.sh, must not feed the C2 traffic)
    reps = [os.path.join(OUT, f"prof_{n}.ncu-rep") for n in ("sweep", "pcg", "sgop")]
    for rep in [r for r in reps if os.path.exists(r)]:
        name = os.path.basename(rep)[5:-8]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        lines = []
        per_launch = []
        for r in rows[2:]:
            kname = r[hdr.index("Kernel Name")].split("(")[0]
            vals = {k: (r[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr}
            lines.append(f"{kname}\n" + "\n".join(f"  {k:60s} {v[0]:>16s} {v[1]}" for k, v in vals.items()))
            def tobytes(k):
                v, u = vals[k]
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
            per_launch.append((kname, tobytes("dram__bytes_read.sum") + tobytes("dram__bytes_write.sum")))
        with open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none, {os.path.basename(rep)}\n\n" + "\n\n".join(lines) + "\n")
        fresh = {}
        for kname, b in per_launch:
            cls = CLASS.get(kname.replace("void ", "").split("<")[0])
            if cls:
                fresh.setdefault(cls, []).append(b)
        for cls, s in fresh.items():  # replaces older samples of the same kernel class
            summary.setdefault(config, {})[cls] = {"dram_bytes_per_launch_samples": s,
                                                   "dram_bytes_per_launch": sum(s) / len(s), "source": f"{tag}_ncu_{name}.txt"}
        print(open(os.path.join(PROF, f"{tag}_ncu_{name}.txt")).read())
    json.dump(summary, open(summary_path, "w"), indent=1)


if __name__ == "__main__":
    os.makedirs(PROF, exist_ok=True)
    tag = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "C2"
    launch_shares(tag)
    full_captures(tag, cfg)
