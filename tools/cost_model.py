"""α-β-γ strong-scaling model of the synchronous DP step (PAPER.md:308-313
"communication complexity O(log(p)) ... approximately C/p + log(p)"), fitted to this round's
measurements and used for LABELLED projections to P = 8 (gpurun offers at most 4 GPUs).

  allreduce:  t_ar(P, bytes) = alpha(P) + bytes * 2(P-1)/P / busbw(P)   (fit per P on the cfg5 sweep)
              alpha(P) = a0 + a1 * log2(P)                              (the paper's O(log p) term)
  step:       T(P) = L + C / P + t_ar(P, grad bytes)                    (L: P-independent latency floor,
                                                                         C: work that divides by P)
L and C are fitted per config to the measured P = 1 and P = 2 steps (fused mode), P = 4 is held
out to test the model, P = 8 is a projection.  Inputs: profiles/<round>_cfg5_P*.jsonl and the
bench lines in profiles/<round>_steps.json.  Output: profiles/<round>_cost_model.md.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "round1"
prof = os.path.join(ROOT, "profiles")

# ---- allreduce fit per P
fits = {}
for P in (2, 4):
    rows = [json.loads(l) for l in open(os.path.join(prof, f"{rnd}_cfg5_P{P}.jsonl"))]
    xs = [r["bytes"] * 2 * (P - 1) / P for r in rows]
    ys = [r["allreduce_us"] * 1e-6 for r in rows]
    n = len(xs)
    mx, my = sum(xs) / n, sum(ys) / n
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
    alpha = min(ys)  # latency floor: the smallest message
    fits[P] = {"alpha_us": alpha * 1e6, "busbw_gbs": 1 / slope / 1e9}
a1 = (fits[4]["alpha_us"] - fits[2]["alpha_us"]) / (math.log2(4) - math.log2(2))
a0 = fits[2]["alpha_us"] - a1
fits[8] = {"alpha_us": a0 + a1 * 3, "busbw_gbs": 725.0}  # 8-rank busbw: B200_PROFILING.md reference (1 GiB)


def t_ar(P, nbytes):
    if P == 1:
        return 0.0
    f = fits[P]
    return f["alpha_us"] * 1e-6 + nbytes * 2 * (P - 1) / P / (f["busbw_gbs"] * 1e9)


steps = json.load(open(os.path.join(prof, f"{rnd}_steps.json")))
L = [f"# α-β-γ strong-scaling model ({rnd}) — projections are labelled, not measured", "",
     "Allreduce fit per P on the cfg5 sweep (ncclAllReduce, fp32): α = smallest-message latency, busbw = least-squares slope.",
     "", "| P | α (µs) | busbw (GB/s) | source |", "|---:|---:|---:|---|"]
for P in (2, 4, 8):
    src = "fit to cfg5 sweep" if P < 8 else f"projection: α = {a0:.1f} + {a1:.1f}·log2 P µs (paper's O(log p)); busbw = 725 GB/s 8-rank reference"
    L.append(f"| {P} | {fits[P]['alpha_us']:.1f} | {fits[P]['busbw_gbs']:.0f} | {src} |")
L += ["", "Step model T(P) = L + C/P + t_ar(P, gradient bytes); L, C fitted to measured P = 1, 2; P = 4 held out.", "",
      "| config | grad MB | FLOP/param/sample | L (µs) | C (µs) | P=4 model (µs) | P=4 measured (µs) | P=8 projection (µs) | E(8) projected |",
      "|---|---:|---:|---:|---:|---:|---:|---:|---:|"]
for cfg, d in steps.items():
    gb = d["grad_bytes"]
    T1, T2 = d["us"]["1"] * 1e-6, d["us"]["2"] * 1e-6
    # T1 = L + C ; T2 = L + C/2 + t_ar(2)
    C = 2 * (T1 - (T2 - t_ar(2, gb)))
    Lat = T1 - C
    T4m = Lat + C / 4 + t_ar(4, gb)
    T8 = Lat + C / 8 + t_ar(8, gb)
    E8 = T1 / (8 * T8)
    ratio = d["flop_per_sample"] / d["params"]
    L.append(f"| {cfg} | {gb / 1e6:.2f} | {ratio:.1f} | {Lat * 1e6:.1f} | {C * 1e6:.1f} | {T4m * 1e6:.1f} | "
             f"{d['us'].get('4', float('nan')):.1f} | {T8 * 1e6:.1f} | {E8:.2f} |")
L += ["", "The paper's qualitative claim (P:464-474): networks with more computation per parameter scale better "
      "(AlexNet worst). Here cfg4 (higher FLOP/param/sample, compute-dominated) scales far better than cfg2, whose step is "
      "a latency floor L that does not divide by P — the strong-scaling limit at B = 512."]
open(os.path.join(prof, f"{rnd}_cost_model.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L))
