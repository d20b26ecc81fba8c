"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

usage: python tools/summarize_profiles.py <tag> [--launches gpurun_out/launches.csv]
                                          [--rep name=gpurun_out/x.ncu-rep ...]
Writes profiles/<tag>_launches.txt (per-kernel share of the ncu launch list) and, per report,
profiles/<tag>_ncu_<name>.txt (duration, DRAM bytes, throughputs, pipe utilisation, top stall
reasons, hottest source lines) plus profiles/traffic.json {kernel_family: dram bytes per launch}
that bench.py reports as roofline.traffic.
"""
import argparse
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path, tag):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised launches): {path}",
           f"# total {tot / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:34s} n={v[0]:5d} total={v[1] / 1e6:9.3f} ms share={100 * v[1] / tot:5.1f}%")
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units, v = r[0], r[1], r[2]
    return {k: (x, u) for k, u, x in zip(h, units, v)}


def report(name, rep, tag):
    m = raw_metrics(rep)

    def g(k):
        x = m.get(k, ("", ""))[0]
        try:
            return float(x.replace(",", ""))
        except ValueError:
            return None

    def unit(k):
        return m.get(k, ("", ""))[1]

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size"]
    lines = [f"# ncu --set full --clock-control none: {os.path.basename(rep)} ({name})"]
    for k in keys:
        lines.append(f"{k:80s} {m.get(k, ('n/a', ''))[0]} {unit(k)}")
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): g(k) for k in m
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(v for v in stalls.values() if v) or 1
    lines.append("# stall reasons (pc sampling, % of samples)")
    for k, v in sorted(stalls.items(), key=lambda kv: -(kv[1] or 0))[:8]:
        lines.append(f"  {k:28s} {100 * (v or 0) / tot:5.1f}")
    hot = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_hot.py"), rep, "12"],
                         capture_output=True, text=True).stdout
    lines.append("# hottest source lines")
    lines += ["  " + ln for ln in hot.splitlines()]
    open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd is not None and wr is not None:
        b = rd * scale.get(unit("dram__bytes_read.sum"), 1) + wr * scale.get(unit("dram__bytes_write.sum"), 1)
        return b
    return None


def report_multi(name, rep, tag, scale_to=1, skip=0, count=None):
    """A report holding several kernels (e.g. the 10 phase kernels of one CG iteration): per-kernel
    duration and DRAM bytes, summed; traffic = sum x scale_to (iterations per solve)."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, units = r[0], r[1]
    idx = {k: i for i, k in enumerate(h)}
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}

    def val(row, k):
        try:
            return float(row[idx[k]].replace(",", "")) * mult.get(units[idx[k]], 1)
        except (KeyError, ValueError):
            return 0.0

    lines = [f"# ncu --set full --clock-control none: {os.path.basename(rep)} ({name}, kernels {skip}.."
             f"{skip + (count if count is not None else len(r) - 2 - skip) - 1} of {len(r) - 2}; caches flushed"
             " between kernels by ncu, so cross-kernel L2 reuse is not credited)"]
    tot_t = tot_b = 0.0
    rows = r[2 + skip:]
    if count is not None:
        rows = rows[:count]
    for row in rows:
        t = val(row, "gpu__time_duration.sum")
        b = val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum")
        dm = row[idx.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0)]
        kname = row[idx["Kernel Name"]].split("(")[0].split("::")[-1] if "Kernel Name" in idx else "?"
        lines.append(f"  {kname:40s} {t * 1e6:9.2f} us  dram {b / 1e6:9.2f} MB  {b / max(t, 1e-12) / 1e9:8.1f} GB/s")
        tot_t += t
        tot_b += b
    lines.append(f"# sum: {tot_t * 1e6:.2f} us, dram {tot_b / 1e6:.2f} MB ({tot_b / max(tot_t, 1e-12) / 1e9:.1f} GB/s); "
                 f"x{scale_to} -> {tot_b * scale_to:.4g} bytes per solve")
    open(os.path.join(PROF, f"{tag}_ncu_{name}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return tot_b * scale_to


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches", default=None)
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--multi", action="append", default=[],
                    help="name=rep=scale[=skip[=count]] (sum over the selected kernels x scale)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in a.rep:
        name, rep = spec.split("=", 1)
        b = report(name, rep, a.tag)
        if b is not None:
            traffic[name] = {"dram_bytes_per_launch": b, "source": f"profiles/{a.tag}_ncu_{name}.txt"}
    for spec in a.multi:
        parts = spec.split("=")
        name, rep, scale = parts[0], parts[1], int(parts[2])
        skip = int(parts[3]) if len(parts) > 3 else 0
        count = int(parts[4]) if len(parts) > 4 else None
        b = report_multi(name, rep, a.tag, scale, skip, count)
        traffic[name] = {"dram_bytes_per_launch": b, "source": f"profiles/{a.tag}_ncu_{name}.txt"}
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
