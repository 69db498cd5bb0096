"""Turn the gpurun_out/ncu/ captures of tools/ncu_capture.sh into the committed profiles/ summaries:

  profiles/<tag>_ncu_traffic.json          DRAM bytes per launch of each scheme's solve kernel (bench `traffic`)
  profiles/<tag>_ncu_traffic_detail.jsonl  read / write / L2 bytes and the (cold, serialised) ncu duration
  profiles/<tag>_launches_summary.txt      per-kernel share of the benchmark step from the launch list
  profiles/<tag>_ncu_wide_vroahk.txt       key sections of the full-set capture of the dominant kernel

    python tools/ncu_summarize.py [--tag r01] [--dir gpurun_out/ncu]
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_metrics_csv(path):
    """ncu --csv output: rows of (kernel, metric, value); returns {kernel: {metric: value}} (first launch)."""
    text = open(path).read()
    start = text.find('"ID"')
    if start < 0:
        return {}
    out = {}
    for row in csv.DictReader(io.StringIO(text[start:])):
        k = row.get("Kernel Name", "")
        d = out.setdefault(k, {})
        name = row.get("Metric Name")
        if name and name not in d:
            try:
                d[name] = (float(row["Metric Value"].replace(",", "")), row.get("Metric Unit", ""))
            except ValueError:
                pass
    return out


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1024, "MB": 1024 ** 2, "GB": 1024 ** 3}
    return v * scale.get(unit, 1)


def to_ms(v, unit):
    return v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                "second": 1e3, "s": 1e3}.get(unit, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--dir", default=os.path.join(ROOT, "gpurun_out", "ncu"))
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    traffic, detail = {}, []
    for sc in ("urk", "grk", "vr-ogrk", "ahk", "vr-oahk"):
        path = os.path.join(a.dir, f"traffic_{sc}.csv")
        if not os.path.exists(path):
            continue
        for kern, m in read_metrics_csv(path).items():
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            l2 = to_bytes(*m["lts__t_bytes.sum"]) if "lts__t_bytes.sum" in m else None
            t = to_ms(*m["gpu__time_duration.sum"])
            traffic[sc] = rd + wr
            detail.append({"scheme": sc, "kernel": kern, "dram_read_B": rd, "dram_write_B": wr, "l2_bytes": l2,
                           "ncu_time_ms_cold": t})
            break
    with open(os.path.join(prof, f"{a.tag}_ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    with open(os.path.join(prof, f"{a.tag}_ncu_traffic_detail.jsonl"), "w") as fh:
        for d in detail:
            fh.write(json.dumps(d) + "\n")
    # launch list of the benchmark command
    lpath = os.path.join(a.dir, "launches.csv")
    if os.path.exists(lpath):
        text = open(lpath).read()
        start = text.find('"ID"')
        tot = defaultdict(float)
        cnt = defaultdict(int)
        for row in csv.DictReader(io.StringIO(text[start:])):
            if row.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = row["Kernel Name"]
            tot[k] += to_ms(float(row["Metric Value"].replace(",", "")), row["Metric Unit"])
            cnt[k] += 1
        s = sum(tot.values())
        lines = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) over",
                 "`python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e` (3 steps incl. warmup + final "
                 "gather step)", "", "  share launches   total_ms  kernel"]
        for k in sorted(tot, key=tot.get, reverse=True):
            lines.append(f"{100 * tot[k] / s:6.2f}% {cnt[k]:8d} {tot[k]:10.3f}  {k}")
        lines.append(f"\n{sum(cnt.values())} launches, {s:.1f} ms total")
        with open(os.path.join(prof, f"{a.tag}_launches_summary.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        subprocess.run(["cp", lpath, os.path.join(prof, f"{a.tag}_launches.csv")])
    # full-set capture of the dominant kernel
    rep = os.path.join(a.dir, "full_vroahk.ncu-rep")
    if os.path.exists(rep):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        keep = ("Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
                "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "No Eligible",
                "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
                "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy")
        lines = ["# ncu --set full --clock-control none, kz_wide_kernel<6> (vr-oahk), cfg2 c64 B=1024 T=50 "
                 "(tools/prof_solve.py)", f"# source: {os.path.relpath(rep, ROOT)}", ""]
        for row in csv.DictReader(io.StringIO(raw)):
            if row.get("Metric Name") in keep:
                lines.append(f"{row['Section Name']} | {row['Metric Name']} | {row['Metric Unit']} | "
                             f"{row['Metric Value']}")
        with open(os.path.join(prof, f"{a.tag}_ncu_wide_vroahk.txt"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
