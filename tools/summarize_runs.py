"""Writes profiles/<round>_cfg5.md and profiles/<round>_scaling.md from gpurun_out/ results."""
import glob, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
go = os.path.join(ROOT, "gpurun_out")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
L = [f"# cfg5 — averaging operator sweep ({rnd})", "",
     "`tools/cfg5_sweep.py` under torchrun, CUDA events on the library stream, max over ranks.",
     "allreduce = `mtx_allreduce_avg(apply_update=0)` (ncclAllReduce sum, fp32); +update = the same call",
     "with the fused average + momentum update (K6); K6 alone on a world-1 context. busbw = algbw·2(P−1)/P.",
     f"K6 GB/s = 20 B/elem ÷ time; HBM reference {peaks['hbm_gbs']} GB/s measured copy (nominal 8000).", ""]
for f in sorted(glob.glob(os.path.join(go, "cfg5_P*.jsonl"))):
    rows = [json.loads(l) for l in open(f)]
    P = rows[0]["P"]
    L += [f"## P = {P}", "", "| elements | bytes | allreduce µs | algbw GB/s | busbw GB/s | allreduce+update µs | K6 µs | K6 GB/s | K6 / measured HBM | note |",
          "|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
    for r in rows:
        L.append(f"| {r['n']:,} | {r['bytes']:,} | {r.get('allreduce_us','')} | {r.get('algbw_gbs','')} | {r.get('busbw_gbs','')} | "
                 f"{r.get('allreduce_update_us','')} | {r['k6_us']} | {r['k6_gbs']} | {r['k6_gbs']/peaks['hbm_gbs']:.3f} | "
                 f"{'L2-resident' if r['l2_resident'] else 'HBM'} |")
    L.append("")
open(os.path.join(ROOT, "profiles", f"{rnd}_cfg5.md"), "w").write("\n".join(L) + "\n")
S = [f"# Strong scaling of the DP step ({rnd})", "", "bench.py lines (device-timed, max over ranks, L2 flushed per step), 3xTF32 tensor cores (fp32-accurate).",
     "Efficiency E(P) = S(P) / (P · S(1)).", "", "| config | P | samples/s | ms/step | per-rank ms (K steps) | E(P) | e2e samples/s |", "|---|---:|---:|---:|---|---:|---:|"]
for cfg in ("cfg2", "cfg3", "cfg4"):
    base = None
    for N in (1, 2, 4, 8):
        f = os.path.join(go, f"scale_{cfg}_N{N}.json")
        if not os.path.exists(f):
            continue
        line = [l for l in open(f) if l.startswith("{")]
        if not line:
            continue
        d = json.loads(line[-1])
        base = base or d["value"]
        S.append(f"| {cfg} | {N} | {d['value']:,.0f} | {d['ms_per_step']:.4f} | {d['per_rank_ms']} | {d['value']/(N*base):.3f} | {d['e2e']['value']:,.0f} |")
S += ["", "8 GPUs: not measurable through gpurun (1, 2 or 4 GPUs per call)."]
open(os.path.join(ROOT, "profiles", f"{rnd}_scaling.md"), "w").write("\n".join(S) + "\n")
print("ok")
