"""One-off box probe: host cores, GPU, NCCL version, TF32/FP32 cuBLAS throughput.

Writes gpurun_out/probe.json. Context numbers only (denominators for the TF32
roofline, which MEASURED_PEAKS.json does not carry)."""
import json, os, subprocess, time
import torch

out = {}
out["nproc"] = os.cpu_count()
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception as e:  # noqa
    out["cpu_model"] = str(e)
out["affinity"] = len(os.sched_getaffinity(0))
out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total", "--format=csv"], capture_output=True, text=True).stdout
out["nccl"] = torch.cuda.nccl.version()
out["torch"] = torch.__version__
p = torch.cuda.get_device_properties(0)
out["sm_count"] = p.multi_processor_count
out["l2"] = p.L2_cache_size


def bench_mm(n, tf32, secs=None, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        torch.mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    if secs is None:
        for _ in range(reps):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); torch.mm(a, b); e.record(); torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        return 2 * n ** 3 / best / 1e12
    t0 = time.time(); cnt = 0
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            torch.mm(a, b)
        cnt += 10
        torch.cuda.synchronize()
    e.record(); torch.cuda.synchronize()
    return 2 * n ** 3 * cnt / (s.elapsed_time(e) / 1e3) / 1e12

out["tf32_tflops_burst_8192"] = bench_mm(8192, True)
out["tf32_tflops_sustained_8192"] = bench_mm(8192, True, secs=4)
out["fp32_tflops_burst_8192"] = bench_mm(8192, False, reps=3)
# shapes of cfg4 (b=8192, 1024x1024)
for (m, n, k) in [(8192, 1024, 1024), (1024, 1024, 8192)]:
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(m, k, device="cuda"); b = torch.randn(k, n, device="cuda")
    for _ in range(5): torch.mm(a, b)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): torch.mm(a, b)
    e.record(); torch.cuda.synchronize()
    out[f"tf32_cublas_{m}x{n}x{k}_us"] = s.elapsed_time(e) / 50 * 1e3
# copy bw
x = torch.empty(1 << 28, device="cuda"); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): y.copy_(x)
e.record(); torch.cuda.synchronize()
out["copy_gbs_fp32_1GiB"] = 2 * x.numel() * 4 * 10 / (s.elapsed_time(e) / 1e3) / 1e9
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
print(json.dumps(out, indent=1))
