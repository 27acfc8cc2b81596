"""Benchmark of the synchronous data-parallel SGD step (BASELINE.json metric:
train samples/sec, device-timed, max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--precision 3xtf32|fp32]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference     # the CPU oracle on the host cores (reference arm)

One "step" = one pass of the whole hot path over one global batch: forward,
softmax-CE, backward, flat-buffer allreduce-sum (NCCL, bucketed, overlapped),
x 1/P and the fused momentum update.  Strong scaling:
the global batch B is fixed and split over the N ranks.
Inputs are seeded synthetic data shaped like the paper's workloads (mtx_synth),
resident in HBM before the timed region.  L2 is flushed (a 256 MiB write)
before every timed step and the flush is outside the events.  Prints ONE JSON
line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}
NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md; 900 nominal)
TF32_PER_BF16 = 1.1 / 2.25  # nominal dense ratio (B200_PROFILING.md table)
FP32_FMA_PER_SM_CLK = 128  # CUDA cores per SM (4 SMSP x 32 lanes), 2 flop per FMA


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        d["_source"] = "measured"
        return d
    d = dict(PEAKS_FALLBACK)
    d["_source"] = "fallback"
    return d


# ----------------------------------------------------------------------------- clocks sampler
class Clocks:
    """Samples SM clock and clock-event reasons through NVML every ~2 ms while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index, self.samples, self.stop_ev = index, [], threading.Event()

    def start(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis else self.index
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.N = N
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.N = None
            self.err = str(e)
            return
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        time.sleep(0.01)

    def _run(self):
        N = self.N
        while not self.stop_ev.is_set():
            try:
                self.samples.append((N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM),
                                     N.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def stop(self):
        self.stop_ev.set()
        if self.N is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled: " + getattr(self, "err", "")]}
        self.t.join(1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        busy = [s for s in self.samples if not (s[1] & 0x1)] or self.samples
        reasons = set()
        for _, r in busy:
            for bit, name in self.REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in busy), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(busy)}


# ----------------------------------------------------------------------------- roofline helpers
def kernel_work(name: str):
    """Algorithmic work per launch from the launch-site name: ('flop'|'byte', amount, bound)."""
    m = re.match(r"(\w+)\[(.*)\]", name)
    if not m:
        return None
    kind, args = m.group(1), dict(kv.split("=") for kv in m.group(2).split(","))
    a = {k: int(v) for k, v in args.items()}
    if kind.startswith("gemm"):
        if kind.startswith("gemm_tc3xf16"):  # 3 fp16 MMAs per product (3xF16 split): vs a third of the f16 peak
            return "flop", 2 * a["M"] * a["N"] * a["K"], "tensor3xf16"
        if kind.startswith("gemm_tc3x"):  # 3 tf32 MMAs per product: tensor work is 3x the algorithmic flops
            return "flop", 2 * a["M"] * a["N"] * a["K"], "tensor3x"
        tensor = kind.startswith("gemm_tc")
        return "flop", 2 * a["M"] * a["N"] * a["K"], "tensor" if tensor else "alu"
    if kind == "colsum":
        return "byte", 4 * a["K"] * a["N"], "hbm"
    if kind == "wgrad_narrow":  # streams A [K x (M-1)] once; dZ is tiny
        return "byte", 4 * a["K"] * (a["M"] - 1 + a["N"]), "hbm"
    if kind == "conv_fwd":  # direct convolution, valid, stride 1: 2 * b * ho^2 * co * ci * k^2 (CUDA-core FMA)
        ho = a["hi"] - a["k"] + 1
        return "flop", 2 * a["rows"] * ho * ho * a["co"] * a["ci"] * a["k"] * a["k"], "alu"
    if kind == "conv_bwd":  # wgrad (+ dgrad): E - 1 = ci * k^2 products per conv output and channel, each
        return "flop", 2 * a["rows"] * a["hc"] * a["hc"] * a["co"] * (a["E"] - 1) * (1 + a["dgrad"]), "alu"
    if kind.startswith("conv_") or kind == "pool_relu_bwd":
        return None
    if kind == "avg_update":
        return "byte", ((20 if a["v"] else 12) + (8 if a.get("planes") else 0)) * a["n"], "hbm"
    if kind == "fused_avg_update":  # NVLink-bound: per direction per GPU, the P-1 peers'
        # gradients of the owned n/P slice come in and the P-1 peers' updated w slices are stored in
        P = a["P"]
        if a.get("push"):  # push protocol: the peers' gradients already landed locally (copy engines, during the
            return "byte", 4 * (a["n"] // P) * (P - 1), "nvlink"  # backward); only the w slices go out
        return "byte", 8 * (a["n"] // P) * (P - 1), "nvlink"
    if kind == "head_softmax_xent":  # read A rows, write dZ_{L-1} (and dZ_L, loss)
        return "byte", 4 * a["rows"] * (a["d"] * (1 + a["dgrad"]) + a["C"] + 1), "hbm"
    if kind == "splitk_reduce":
        return "byte", 4 * a["M"] * a["N"] * (a["splits"] + 1), "hbm"
    if kind == "loss_reduce":
        return "byte", 4 * a["n"], "hbm"
    return None


def roofline(timing: dict, pk: dict, sm_mhz: float | None, steps: int, config: str):
    """Dominant kernel launch (one kernel at one shape/plan, by total device time per step) -> achieved / peak.

    Each kernel's event pair inside the timing graph also spans the graph's per-node launch
    latency; the timing graph brackets an empty kernel the same way ("launch_overhead") and that
    per-launch overhead is subtracted from every launch (clamped at 10% of the raw time)."""
    cal = timing.pop("launch_overhead[calibration]", None)
    over_ms = cal[0] / cal[1] if cal and cal[1] else 0.0
    timing = {k: (max(ms - over_ms * cnt, 0.1 * ms), cnt) for k, (ms, cnt) in timing.items()}
    groups = {}
    for name, (ms, cnt) in timing.items():
        w = kernel_work(name)
        base = name.split("[")[0]
        g = groups.setdefault(base, {"ms": 0.0, "cnt": 0, "work": 0.0, "unit": None, "bound": None})
        g["ms"] += ms
        g["cnt"] += cnt
        if w:
            g["work"] += w[1] * cnt
            g["unit"], g["bound"] = w[0], w[2]
    total = sum(g["ms"] for g in groups.values())
    # the dominant LAUNCH (kernel + shape): a class mixes shapes whose rates differ (cfg4's 28-row weight gradient
    # runs the same kernel as the 1024-row ones at a fraction of the rate); kernels without algorithmic work
    # (peer_barrier: a cross-GPU wait) are not roofline candidates
    launches = {}
    for name, (ms, cnt) in timing.items():
        w = kernel_work(name)
        if w:
            launches[name] = {"ms": ms, "cnt": cnt, "work": w[1] * cnt, "unit": w[0], "bound": w[2]}
    if launches:
        top_launch, top = max(launches.items(), key=lambda kv: kv[1]["ms"])
        top_name = top_launch.split("[")[0]
    else:
        top_name, top = max(groups.items(), key=lambda kv: kv[1]["ms"])
        top_launch = top_name
    per_launch_s = top["ms"] / 1e3 / top["cnt"]
    per_launch_work = top["work"] / top["cnt"]
    # every kernel of the timing pass runs alone (serialised graph): the burst peaks apply
    if top["bound"] == "hbm":
        achieved = per_launch_work / per_launch_s / 1e9
        peak, unit = pk["hbm_gbs"], "GB/s"
    elif top["bound"] == "nvlink":
        achieved = per_launch_work / per_launch_s / 1e9
        peak, unit = NVLINK_GBS, "GB/s"
    elif top["bound"] == "tensor":
        achieved = per_launch_work / per_launch_s / 1e12
        peak, unit = pk["bf16_tflops"] * TF32_PER_BF16, "TFLOP/s"
    elif top["bound"] == "tensor3x":  # fp32-equivalent flops vs one third of the tf32 peak
        achieved = per_launch_work / per_launch_s / 1e12
        peak, unit = pk["bf16_tflops"] * TF32_PER_BF16 / 3, "TFLOP/s"
        top["bound"] = "tensor"
    elif top["bound"] == "tensor3xf16":  # fp32-equivalent flops vs one third of the f16 (= bf16) peak
        achieved = per_launch_work / per_launch_s / 1e12
        peak, unit = pk["bf16_tflops"] / 3, "TFLOP/s"
        top["bound"] = "tensor"
    else:  # fp32 CUDA-core FMA peak at the clock observed under load
        achieved = per_launch_work / per_launch_s / 1e12
        clk = sm_mhz or pk.get("sm_max_mhz", 1965.0)
        peak, unit = 148 * FP32_FMA_PER_SM_CLK * 2 * clk * 1e6 / 1e12, "TFLOP/s"
    # DRAM bytes per launch of the same kernel from the committed ncu --set full capture
    # (profiles/ncu_traffic.json, written by tools/ncu_summary.py), averaged over its captured launches
    # the tensor-core GEMM's template is <N tile, 3xTF32>: take the N tile of the group's longest launch
    longest = top_launch
    bn = re.search(r"bn=(\d+)", longest)
    bn = bn.group(1) if bn else "128"
    pr = re.search(r"pair=(\d)", longest)
    pair = int(pr.group(1)) if pr else 0
    la = dict(kv.split("=") for kv in re.match(r"\w+\[(.*)\]", longest).group(1).split(",")) if "[" in longest else {}
    sp, cl = int(la.get("splits", 1)), int(la.get("cluster", 0))
    f16 = top_name.startswith("gemm_tc3xf16")
    # epilogue mode of the kernel the launch ran (gemm_tc.cu launch_variant): CLU = split-K cluster, PART = split-K
    # partials (unpaired), FAST = 3xF16 pair with every tile whole (M % 256, N % 128; lean or fp32-only output)
    clu = 1 if cl and (not pair or f16) else 0
    part = 1 if sp > 1 and not cl and not pair else 0
    fast = 1 if f16 and pair and sp == 1 and not cl and int(la.get("M", 1)) % 256 == 0 and int(la.get("N", 1)) % 128 == 0 \
        else 0
    # <BN, 3x, PAIR, MASK, F16, FAST, CLU, PART>
    tpl = f"{bn}, {{}}, {pair}, {1 if '_dgrad' in longest else 0}, {{}}, {fast}, {clu}, {part}"
    ncu_kernel = {"gemm_tc3xf16": f"tc_gemm_kernel<{tpl.format(1, 1)}>", "gemm_tc3x": f"tc_gemm_kernel<{tpl.format(1, 0)}>",
                  "gemm_tc": f"tc_gemm_kernel<{tpl.format(0, 0)}>",
                  "avg_update": "avg_update_kernel<1>", "fused_avg_update": "fused_avg_update_kernel", "head_softmax_xent": "head_kernel",
                  "colsum": "colsum_kernel", "splitk_reduce": "splitk_reduce_kernel", "conv_bwd": "conv_bwd_kernel",
                  "conv_fwd": "conv_fwd_kernel"}
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    key = next((v for k, v in ncu_kernel.items() if top_name.startswith(k)), None)
    if os.path.exists(tp) and key:
        tj = json.load(open(tp))
        hit = next((k for k in tj if k == f"{config}:{key}" or k.startswith(f"{config}:{key}<")
                    or k.startswith(f"{config}:{key}(")), None)
        if hit:
            traffic = tj[hit]
            meta = tj.get("_meta", {}).get(config, {})
            traffic_src = f"profiles/ncu_traffic.json [{hit}] from {meta.get('capture', 'ncu --set full')}" \
                          f" at commit {meta.get('commit', '?')}"
    return {"kernel": top_name, "launch": top_launch, "bound": top["bound"], "achieved": round(achieved, 3),
            "peak": round(peak, 1),
            "unit": unit, "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
            "peak_kind": {"GB/s": "measured copy" if top["bound"] == "hbm" else "measured NVLink peer copy per direction",
                          "TFLOP/s": ("measured bf16 burst (= f16 dense) / 3 (3xF16: three f16 MMAs per product)"
                                      if top_name.startswith("gemm_tc3xf16") else
                                      "measured bf16 burst x tf32/bf16 nominal ratio" +
                                      (" / 3 (3xTF32)" if top_name.startswith("gemm_tc3x") else ""))}.get(unit),
            "work_per_launch": per_launch_work, "launch_us": round(per_launch_s * 1e6, 3),
            "share_of_kernel_time": round(top["ms"] / total, 3),  # this launch shape's share of the step's kernel time
            "launch_overhead_us_subtracted": round(over_ms * 1e3, 3),
            "breakdown_us_per_step": {k: round(g["ms"] * 1e3 / steps, 2) for k, g in
                                      sorted(groups.items(), key=lambda kv: -kv[1]["ms"])},
            # every distinct launch of the step (name carries the shape / plan), overhead-corrected
            "launches_us_per_step": {k: round(ms * 1e3 / steps, 2) for k, (ms, cnt) in
                                     sorted(timing.items(), key=lambda kv: -kv[1][0])}}


# ----------------------------------------------------------------------------- CPU oracle baseline
def host_cpu():
    """(nproc, CPU model) of the host running the oracle."""
    model = "unknown"
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def cpu_oracle(cfg: dict, budget_s: float, X, y):
    """The oracle as it stands (plain C, f64) on a bounded sample of the workload, as SURVEY.md §8(d)
    plans it: the oracle's own DP(T) simulation -- T = the host's cores (a power of two dividing B,
    <= 64) simulated ranks, one host thread per rank for the local gradients (O5-O7, ctypes releases the
    GIL), then the single-threaded ascending-rank fold (O9) and update (O10-O11) -- at a global batch of
    T * b_s rows per step (the per-sample cost of an MLP/CNN step does not depend on the batch), for
    about budget_s seconds.  By I1 its result is the sequential SGD step's."""
    from concurrent.futures import ThreadPoolExecutor

    import numpy as np

    import oracle
    nproc, model = host_cpu()
    T = 1
    while T * 2 <= min(nproc, 64) and cfg["B"] % (T * 2) == 0:
        T *= 2
    net = oracle.Net.from_cfg(cfg)
    w = oracle.init_params(net, 42).astype(np.float64)
    v = np.zeros_like(w)
    # rows per simulated rank per step: about 1/8 of budget_s per step, from a one-row probe
    t0 = time.perf_counter()
    oracle.local_grad(net, w, X, y, 1, 0, 0, 1)
    per_row = max(time.perf_counter() - t0, 1e-6)
    b_s = int(max(1, min(cfg["B"] // T, budget_s / 8 / per_row)))
    Bs = T * b_s
    pool = ThreadPoolExecutor(T)
    t0 = time.perf_counter()
    steps = 0
    while True:
        res = list(pool.map(lambda r: oracle.local_grad(net, w, X, y, Bs, steps, r, T), range(T)))
        G = oracle.fold(np.stack([g for g, _ in res]))
        oracle.avg_update(G, w, v, T, cfg["lr"], cfg["mu"])
        steps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    pool.shutdown()
    return {"value": round(Bs * steps / dt, 3), "unit": "samples/s", "cores": T, "kind": "oracle",
            "nproc": nproc, "cpu_model": model,
            "sample": f"{steps} DP({T}) SGD steps of {cfg['name']} at a global batch of {Bs} rows ({b_s} per "
                      f"simulated rank, same per-sample work as B={cfg['B']}), oracle f64 (gcc -O2, no contraction), "
                      f"{T} host threads for the local gradients, fold + update single-threaded, {dt:.1f} s"}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    # cfg4 (the largest config; the north_star's scaling target is quoted on it)
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "3xtf32", "3xf16"])
    ap.add_argument("--impl", default="mtx", choices=["mtx", "reference"])
    ap.add_argument("--bucket-mb", type=float, default=1.0)
    ap.add_argument("--reduce", default="fused", choices=["nccl", "ordered", "fused", "layerwise", "zero1"],
                    help="gradient allreduce (N > 1): NCCL per bucket, ORDERED test mode, or the averaging "
                         "operator fused with its collective over NVLink peer memory")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: >= 3 warm-up steps"

    import numpy as np

    import mtx_synth as S
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(S.CONFIGS[args.config])
    cfg["name"] = args.config
    metric = "train samples/sec (device-timed, max over ranks)"

    if args.impl == "reference":
        if rank != 0:
            return
        X, y = S.dataset(cfg, n=min(cfg["n"], 100_000))
        cb = cpu_oracle(cfg, max(2.0, min(args.cpu_budget, 10.0)), X, y)
        line = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": "samples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(cfg["B"] / cb["value"] * 1e3, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": run_config(args, cfg, args.gpus),
                "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    # stdout must carry exactly one JSON line: NCCL logs to stdout (its version banner prints at
    # every level from VERSION up, WARN included), so its log goes to stderr
    if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION"):
        os.environ["NCCL_DEBUG"] = "WARN"
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch
    import torch.distributed as dist

    import paper_1704_04560_b200 as P
    from paper_1704_04560_b200 import mtx
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tc_ok = "tcgen05" in mtx.mtx_build_info()
    # auto: the fastest fp32-tier tensor-core mode measured for the workload: 3xF16 for cfg4's large
    # GEMMs; 3xTF32 for the small latency-bound ones of cfg1-3 (the 3xF16 parameter quantize does not pay there)
    auto = (P.MTX_3XF16 if args.config == "cfg4" else P.MTX_3XTF32) if tc_ok else P.MTX_FP32
    prec = {"fp32": P.MTX_FP32, "3xtf32": P.MTX_3XTF32, "3xf16": P.MTX_3XF16}.get(args.precision, auto)
    uid = P.nccl_uid_broadcast(rank, world)
    X, y = S.dataset(cfg)
    reduce = {"nccl": P.MTX_REDUCE_NCCL, "ordered": P.MTX_REDUCE_ORDERED, "fused": P.MTX_REDUCE_FUSED,
              "layerwise": P.MTX_REDUCE_LAYERWISE, "zero1": P.MTX_REDUCE_ZERO1}[args.reduce]
    rep = P.Replica(cfg, rank=rank, world=world, uid=uid, device=local, precision=prec,
                    bucket_bytes=int(args.bucket_mb * (1 << 20)), reduce=reduce if world > 1 else P.MTX_REDUCE_NCCL)
    rep.bcast()
    rep.shard(X, y)
    s = rep.stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        rep.step()
    barrier()
    clocks = Clocks(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    # head start: the stream spins (outside every event pair) while the host enqueues all K steps,
    # so host issue jitter on one rank cannot show up as peer wait inside another rank's step.  The spin
    # must still be running when the enqueue loop ends (checked; else retried with a longer spin).
    spin_ms = min(0.2 * args.steps + 2.0, 100.0)
    for attempt in range(4):
        barrier()
        spun = torch.cuda.Event()
        with torch.cuda.stream(s):
            torch.cuda._sleep(int(spin_ms * 2.0e6))
            spun.record(s)
        for k in range(args.steps):
            with torch.cuda.stream(s):
                flush.fill_(k & 0xFF)  # evict L2 (126 MB) before every timed step; outside the events
                ev[k][0].record(s)
            rep.step()
            with torch.cuda.stream(s):
                ev[k][1].record(s)
        covered = not spun.query()  # the GPU was still spinning when the host finished enqueueing
        if world > 1:
            cv = torch.tensor([1 if covered else 0])
            dist.all_reduce(cv, op=dist.ReduceOp.MIN)
            covered = bool(cv[0])
        barrier()
        if covered:
            break
        spin_ms *= 3
    clk = clocks.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    loss = mtx.mtx_train_step(rep.ctx, rep.step_idx, True, rep.s)
    rep.step_idx += 1
    t_all = [t_ms]
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, tt)
        t_all = [float(g[0]) for g in gathered]
    t_max = max(t_all)
    value = cfg["B"] * args.steps / (t_max / 1e3)
    launches = mtx.mtx_launches_per_step(rep.ctx)

    # kernel timing pass (eager launches bracketed by CUDA events on the launching stream)
    mtx.mtx_set_timing(rep.ctx, True)
    for _ in range(2):  # capture + upload of the timing graph happen in these replays: not timed
        rep.step()
    mtx.mtx_read_timing(rep.ctx, reset=True)
    for k in range(args.steps):
        with torch.cuda.stream(s):
            flush.fill_(k & 0xFF)
        rep.step()
    timing = mtx.mtx_read_timing(rep.ctx, reset=True)
    mtx.mtx_set_timing(rep.ctx, False)
    pk = peaks()
    roof = roofline(timing, pk, clk.get("sm_mhz"), args.steps, args.config)
    roof["peak_source"] = pk["_source"]

    # end-to-end through the public API with HOST inputs: per step H2D of the rank's rows from
    # pinned memory, the step, D2H of the loss (mtx_train_step_host)
    n = cfg["n"]
    d = X.reshape(n, -1).shape[1]
    Xh = torch.from_numpy(np.concatenate([X.reshape(n, -1), X.reshape(n, -1)[: cfg["B"]]])).pin_memory()
    yh = torch.from_numpy(np.concatenate([y, y[: cfg["B"]]])).pin_memory()
    b = cfg["B"] // world
    # the pipelined user path (mtx_train_step_host_async): step t+1's host->device copy overlaps step
    # t's compute; every step's loss is copied back to host memory; one mtx_sync at the end
    # each step's rows: pinned host addresses computed before the timed loop (the loop is then only
    # the C calls a data-reader loop would make)
    xp0, yp0 = Xh.data_ptr(), yh.data_ptr()
    ptrs = [(xp0 + 4 * d * ((k * cfg["B"]) % n + rank * b), yp0 + 4 * ((k * cfg["B"]) % n + rank * b))
            for k in range(max(3, args.steps))]
    for k in range(3):
        mtx.mtx_train_step_host_async(rep.ctx, ptrs[k][0], ptrs[k][1], rep.s)
    rep.sync_host()
    barrier()
    t0 = time.perf_counter()
    for k in range(args.steps):
        mtx.mtx_train_step_host_async(rep.ctx, ptrs[k][0], ptrs[k][1], rep.s)
    e2e_loss = rep.sync_host()
    t_e2e = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([t_e2e], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt[0])
    e2e = {"value": round(cfg["B"] * args.steps / t_e2e, 1), "unit": "samples/s",
           "h2d_bytes_per_step": b * (4 * d + 4), "d2h_bytes_per_step": 4,
           "api": "mtx_train_step_host_async x K + mtx_sync (host timer around the loop)",
           "final_loss": round(float(e2e_loss), 6)}

    # invariant I2 on the hardware: every replica's parameters and velocity bit-identical after the run
    dig = rep.digest()
    digs = [dig]
    if world > 1:
        dd = torch.tensor([dig & 0x7FFFFFFFFFFFFFFF, dig >> 63], dtype=torch.int64)
        outs = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(outs, dd)
        digs = [int(o[0]) | (int(o[1]) << 63) for o in outs]

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_oracle(cfg, args.cpu_budget, X[:100_000], y[:100_000])
    if rank == 0:
        line = {"metric": metric, "value": round(value, 1), "unit": "samples/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 5),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": {P.MTX_TF32: "tf32", P.MTX_3XTF32: "f32 (3xtf32 tensor cores)",
                          P.MTX_3XF16: "f32 (3xf16 scaled split, tensor cores)"}.get(prec, "f32"),
                "data": "synthetic",
                "config": run_config(args, cfg, world), "engine": mtx.mtx_build_info(),
                "per_rank_ms": [round(t, 3) for t in t_all], "final_loss": loss,
                "replicas_bit_identical": len(set(digs)) == 1, "param_digest": f"{digs[0]:016x}",
                "head_start": {"spin_ms": spin_ms, "covered_enqueue": covered},
                "gpu_launches": launches * args.steps, "launches_per_step": launches,
                "clocks": clk, "roofline": roof, "cpu_baseline": cb, "e2e": e2e}
        print(json.dumps(line), flush=True)
    rep.close()
    if world > 1:
        dist.destroy_process_group()


def run_config(args, cfg, world):
    """The workload both arms report (identical dicts: the driver compares them)."""
    return {"workload": f"{args.config}: {desc(cfg)}", "global_batch": cfg["B"], "local_batch": cfg["B"] // world,
            "parallelism": f"dp{world}", "bucket_mb": args.bucket_mb,
            "reduce": args.reduce if world > 1 else "none (P=1)",
            "l2": "flushed (256 MiB write) before every timed step"}


def desc(cfg):
    if cfg["kind"] == "mlp":
        return f"MLP {'-'.join(map(str, cfg['dims']))}, {cfg['data']}-shaped n={cfg['n']}, B={cfg['B']}, lr={cfg['lr']}, mu={cfg['mu']}"
    return f"LeNet CNN {cfg['in_hwc']}, {cfg['data']}-shaped n={cfg['n']}, B={cfg['B']}, lr={cfg['lr']}, mu={cfg['mu']}"


if __name__ == "__main__":
    main()
