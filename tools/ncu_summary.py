"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/ncu_summary.py <tag> <config> [round]

Reads gpurun_out/launches_<tag>.csv (gpu__time_duration.sum launch list) and
gpurun_out/prof_<tag>.ncu-rep (--set full capture) and writes
profiles/<round>_<tag>.md plus merges per-kernel DRAM traffic per launch into
profiles/ncu_traffic.json (keyed "<config>:<kernel>") for bench.py's roofline.
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, config = sys.argv[1], sys.argv[2]
rnd = sys.argv[3] if len(sys.argv) > 3 else "round1"
out_md = os.path.join(ROOT, "profiles", f"{rnd}_{tag}.md")
lines = [f"# ncu summary — {tag} ({config}), {rnd}", ""]


def short(name):
    name = re.sub(r"\((?!int|bool).*", "", name)  # drop the argument list, keep template args
    name = re.sub(r"^(void )?.*?::(?=[a-z_0-9]+_kernel)", "", name.strip())
    name = name.replace("(int)", "").replace("(bool)", "").replace("true", "1").replace("false", "0")
    return name.strip()


# ---- launch list
launch_csv = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(launch_csv):
    rows = list(csv.reader(open(launch_csv)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        us = v / 1000 if unit.startswith("n") else (v * 1000 if unit.startswith("m") else v)
        a = agg.setdefault(short(d["Kernel Name"]), [0, 0.0])
        a[0] += 1
        a[1] += us
    agg.pop("spin_kernel", None)  # bench's timing-pass spin (not part of a step)
    tot = sum(a[1] for a in agg.values())
    lines += ["## Launch list (ncu `gpu__time_duration.sum`, `--clock-control none`; cold-cache, serialised)", "",
              "Share of device time over all captured launches of the bench command (the spin kernel of the",
              "timing pass excluded). Compare shares with bench.py's roofline, not absolutes.", "",
              "| kernel | launches | total µs | mean µs | share |", "|---|---:|---:|---:|---:|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {t / n:.2f} | {t / tot:.3f} |")
    lines.append("")

# ---- full capture
rep = os.path.join(ROOT, "gpurun_out", f"prof_{tag}.ncu-rep")
traffic = {}
if os.path.exists(rep):
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed",
               "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
               "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
               "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    idx = {k: i for i, k in enumerate(h)}
    lines += ["## `--set full` capture (per launch)", "",
              "| kernel | grid×block | regs | µs | DRAM read MB | DRAM write MB | DRAM % | tensor pipe % | SM % | L1/TEX % |",
              "|---|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
    per = collections.defaultdict(list)
    for row in r[2:]:
        g = lambda m: row[idx[m]] if m in idx else ""
        name = short(g("Kernel Name"))

        def mb(m):
            u = units[idx[m]]
            v = float(g(m).replace(",", "") or 0)
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(u, 1)
            return v * scale
        rd, wr = mb("dram__bytes_read.sum"), mb("dram__bytes_write.sum")
        tu = units[idx["gpu__time_duration.sum"]]
        t = float(g("gpu__time_duration.sum").replace(",", ""))
        t = t / 1000 if tu.startswith("n") else (t * 1000 if tu.startswith("m") else t)
        lines.append(f"| `{name}` | {g('launch__grid_size')}×{g('launch__block_size')} | {g('launch__registers_per_thread')} | "
                     f"{t:.2f} | {rd:.2f} | {wr:.2f} | {g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed')} | "
                     f"{g('sm__throughput.avg.pct_of_peak_sustained_elapsed')} | {g('l1tex__throughput.avg.pct_of_peak_sustained_elapsed')} |")
        per[name].append((rd + wr) * 1e6)
    for k, v in per.items():
        traffic[f"{config}:{k}"] = sum(v) / len(v)
    lines.append("")
open(out_md, "w").write("\n".join(lines) + "\n")
tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
old = json.load(open(tp)) if os.path.exists(tp) else {}
for k in [k for k in old if k.startswith(f"{config}:")]:  # a new capture of this config replaces the old one
    del old[k]
old.update(traffic)
if traffic:  # provenance of this config's capture, read back by bench.py (traffic_source)
    head = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"], capture_output=True, text=True).stdout.strip()
    old.setdefault("_meta", {})[config] = {"capture": f"gpurun_out/prof_{tag}.ncu-rep (ncu --set full, summary "
                                                      f"profiles/{rnd}_{tag}.md)", "commit": head}
json.dump(old, open(tp, "w"), indent=1, sort_keys=True)
print(out_md)
