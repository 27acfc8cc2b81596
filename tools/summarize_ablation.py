"""profiles/<round>_reduce_modes.md from gpurun_out/abl_*.json (reduce-mode ablation)."""
import glob, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
rows = {}
for f in glob.glob(os.path.join(ROOT, "gpurun_out", "abl_*.json")):
    lines = [l for l in open(f) if l.startswith("{")]
    if not lines:
        continue
    d = json.loads(lines[-1])
    _, cfg, n, mode = os.path.basename(f)[:-5].split("_")
    rows[(cfg, int(n[1:]), mode)] = d
L = [f"# Gradient-reduction modes, ablation ({rnd})", "",
     "bench.py lines (3xTF32 step, device-timed, max over ranks, L2 flushed per step). Modes (include/mtx.h):",
     "`nccl` = flat buffer, reverse-layer 1 MiB buckets, ncclAllReduce per bucket overlapped with the backward, then K6;",
     "`fused` = the averaging operator fused with its collective over NVLink peer memory (one kernel + 2 flag barriers);",
     "`layerwise` = the paper's design (P:304-306): one ncclAllReduce per variable in canonical order after the backward;",
     "`zero1` = ncclReduceScatter, update of the 1/P shard, ncclAllGather of w, v (and G);",
     "`ordered` = test mode: allgather of every rank's buckets + an ascending-rank left fold (the oracle's order).", "",
     "| config | P | mode | µs/step | samples/s | vs fused |", "|---|---:|---|---:|---:|---:|"]
for cfg in ("cfg2", "cfg4"):
    for n in (2, 4):
        base = rows.get((cfg, n, "fused"))
        for mode in ("nccl", "fused", "layerwise", "zero1", "ordered"):
            d = rows.get((cfg, n, mode))
            if not d:
                continue
            rel = d["ms_per_step"] / base["ms_per_step"] if base else float("nan")
            L.append(f"| {cfg} | {n} | {mode} | {d['ms_per_step']*1000:.1f} | {d['value']:,.0f} | {rel:.2f}× |")
open(os.path.join(ROOT, "profiles", f"{rnd}_reduce_modes.md"), "w").write("\n".join(L) + "\n")
print("ok")
