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
import sys
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


# (capture, title, kernel symbol substring for the line map, output suffix)
FULL_SETS = [
    ("full_vroahk", "kz_wide_kernel<6> (vr-oahk), cfg2 c64 B=1024 T=50", "kz_wide_kernelILi6E", "ncu_wide_vroahk"),
    ("full_wide_grk", "kz_wide_kernel<4> (grk), cfg2 c64 B=1024 T=50", "kz_wide_kernelILi4E", "ncu_wide_grk"),
    ("full_wide_ahk", "kz_wide_kernel<5> (ahk), cfg2 c64 B=1024 T=50", "kz_wide_kernelILi5E", "ncu_wide_ahk"),
    ("full_cfg3_vr-oahk", "kz_cluster_kernel<6,16> (vr-oahk), cfg3 c64 B=128 T=20", "kz_cluster_kernelILi6ELi16",
     "ncu_cluster_cfg3_vroahk"),
    ("full_cfg5_ahk", "kz_cluster_kernel<5,32> (ahk), cfg5 c64 B=64 T=20", "kz_cluster_kernelILi5ELi32",
     "ncu_cluster_cfg5_ahk"),
]
KEEP = ("Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "L1/TEX Hit Rate", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy")


def full_summary(rep, title, ksub):
    """Details-page metrics, stall samples grouped by straight-line SASS blocks (same execution count: one
    block is one loop body / phase), and the hottest source lines (tools/sass_lines.py, current build)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    lines = [f"# ncu --set full --clock-control none --import-source on, {title} (tools/prof_solve.py)",
             f"# source: {os.path.relpath(rep, ROOT)}", ""]
    for row in csv.DictReader(io.StringIO(raw)):
        if row.get("Metric Name") in KEEP:
            lines.append(f"{row['Section Name']} | {row['Metric Name']} | {row['Metric Unit']} | "
                         f"{row['Metric Value']}")
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    if len(rows) > 2:
        hdr = rows[1]
        col = {n: i for i, n in enumerate(hdr)}
        data = rows[2:]
        S = "Warp Stall Sampling (All Samples)"
        tot = sum(float(r[col[S]] or 0) for r in data) or 1.0
        base = int(data[0][col["Address"]], 16)
        blocks = []
        for r in data:
            ex = int(float(r[col["Instructions Executed"]] or 0))
            ad = int(r[col["Address"]], 16) - base
            st = float(r[col[S]] or 0)
            if blocks and blocks[-1][2] == ex:
                blocks[-1][1] = ad
                blocks[-1][3] += st
                blocks[-1][4] += 1
            else:
                blocks.append([ad, ad, ex, st, 1])
        lines += ["", "## stall samples by SASS block (contiguous instructions with one execution count)",
                  "   offsets            executions  instrs  stall%"]
        for b in sorted(blocks, key=lambda x: -x[3])[:14]:
            lines.append(f"  {b[0]:#07x}-{b[1]:#07x} {b[2]:12d} {b[4]:7d}  {100 * b[3] / tot:5.1f}")
        tmp = rep + ".sass.csv"
        with open(tmp, "w") as fh:
            fh.write(sass)
        lib = os.path.join(ROOT, "paper_2501_10689_b200", "libkaczmarz_b200.so")
        hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_lines.py"), lib, ksub, tmp, "15"],
                             capture_output=True, text=True).stdout
        lines += ["", "## hottest source lines (tools/sass_lines.py against the build that was profiled)", hot.rstrip()]
    return "\n".join(lines)


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
    # shared-memory traffic measured by ncu for the wide-kernel captures (cfg2, B=1024, T=50): the bench's
    # roofline.smem_ncu scales it to its own T (bytes are per iteration; setup is <1%)
    smem = {}
    for sc, rep_name in (("vr-oahk", "full_vroahk"), ("grk", "full_wide_grk"), ("ahk", "full_wide_ahk")):
        rep = os.path.join(a.dir, rep_name + ".ncu-rep")
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        if len(rows) < 3:
            continue
        m = dict(zip(rows[0], rows[2]))
        wf = float(m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"].replace(",", ""))
        smem[sc] = {"capture": rep_name, "B": 1024, "T": 50,
                    "shared_wavefronts": wf, "shared_bytes": wf * 128.0,
                    "shared_bytes_per_iteration": wf * 128.0 / 50,
                    "excessive_wavefronts": float(m.get("derived__memory_l1_wavefronts_shared_excessive", "0").replace(",", "")),
                    "pct_of_peak_sustained_elapsed": float(
                        m["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]),
                    "duration_ms": float(m["gpu__time_duration.sum"].replace(",", ""))}
    if smem:
        with open(os.path.join(prof, f"{a.tag}_ncu_smem.json"), "w") as fh:
            json.dump(smem, fh, indent=1)
    # full-set captures: key metrics, stall samples by straight-line SASS block, hottest source lines
    for rep_name, title, ksub, out in FULL_SETS:
        rep = os.path.join(a.dir, rep_name + ".ncu-rep")
        if os.path.exists(rep):
            with open(os.path.join(prof, f"{a.tag}_{out}.txt"), "w") as fh:
                fh.write(full_summary(rep, title, ksub) + "\n")
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
