"""bench.py host logic on CPU: the roofline's work model per launch name, and the reference arm's
JSON line (the oracle timed on host cores)."""
import importlib.util
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.parametrize("name,want", [
    # 2 M N K flops; 3xTF32 is the same algorithmic work against a third of the tensor peak
    ("gemm_tc3x_fwd[M=512,N=512,K=784,splits=4,cluster=1,pair=0,bn=64]", ("flop", 2 * 512 * 512 * 784, "tensor3x")),
    ("gemm_tc_wgrad[M=784,N=512,K=512,splits=4,cluster=1,pair=0,bn=128]", ("flop", 2 * 784 * 512 * 512, "tensor")),
    ("gemm_simt_fwd[M=64,N=128,K=784,splits=1]", ("flop", 2 * 64 * 128 * 784, "alu")),
    # HBM kernels: bytes they must move
    ("avg_update[n=1000,v=1,planes=1]", ("byte", 28 * 1000, "hbm")),
    ("avg_update[n=1000,v=0,planes=0]", ("byte", 12 * 1000, "hbm")),
    # NVLink bytes per direction per GPU: (P-1) peer gradient slices of n/P floats in, (P-1) w slices in
    ("fused_avg_update[n=669760,P=2,v=1]", ("byte", 8 * 334880, "nvlink")),
    ("fused_avg_update[n=1000,P=4,v=0]", ("byte", 8 * 250 * 3, "nvlink")),
    ("colsum[K=512,N=512,splits=8]", ("byte", 4 * 512 * 512, "hbm")),
    ("head_softmax_xent[rows=512,d=512,C=10,dgrad=1]", ("byte", 4 * 512 * (2 * 512 + 11), "hbm")),
    # LeNet: conv1 32x32x3 -> 28x28x6 (k = 5); conv2 backward 10x10x16 outputs, 6*25 inputs each
    ("conv_fwd[rows=1024,hi=32,ci=3,k=5,co=6,spc=1]", ("flop", 2 * 1024 * 28 * 28 * 6 * 3 * 25, "alu")),
    ("conv_bwd[rows=1024,hc=10,E=151,co=16,dgrad=1,ctas=256]", ("flop", 2 * 2 * 1024 * 100 * 16 * 150, "alu")),
    ("conv_bwd[rows=1024,hc=28,E=76,co=6,dgrad=0,ctas=256]", ("flop", 2 * 1024 * 784 * 6 * 75, "alu")),
])
def test_kernel_work_model(name, want):
    assert _bench().kernel_work(name) == want


def test_kernel_work_unknown_names():
    b = _bench()
    assert b.kernel_work("empty_kernel") is None
    assert b.kernel_work("pool_relu_bwd[rows=4,c=6]") is None
    assert b.kernel_work("peer_barrier[P=2]") is None


def test_roofline_skips_kernels_without_work():
    """A cross-GPU barrier can take the most device time (it waits for the slowest rank); the
    roofline reports the dominant kernel that does algorithmic work."""
    b = _bench()
    timing = {"peer_barrier[P=2]": (0.30, 20),
              "gemm_tc3x_fwd[M=256,N=512,K=784,splits=4,cluster=1,pair=0,bn=32]": (0.16, 20),
              "fused_avg_update[n=669760,P=2,v=1]": (0.18, 20)}
    pk = {"hbm_gbs": 6550.0, "bf16_tflops": 1650.0, "bf16_tflops_sustained": 1500.0}
    r = b.roofline(timing, pk, 1965.0, 20, "cfg2")
    assert r["kernel"] == "fused_avg_update" and r["bound"] == "nvlink" and r["unit"] == "GB/s"
    assert abs(r["achieved"] - 8 * 334880 / (0.18e-3 / 20) / 1e9) < 1e-2 and r["peak"] == 770.0
    assert "peer_barrier" in r["breakdown_us_per_step"]


def test_roofline_takes_the_dominant_launch_not_the_class():
    """cfg4's 28-row weight gradient shares the kernel class with the 1024-row ones at a fraction of their rate:
    the roofline is the launch (kernel + shape) with the most device time, rated on its own work."""
    b = _bench()
    big = "gemm_tc3xf16_wgrad[M=1024,N=1024,K=8192,splits=2,cluster=1,pair=1,bn=128]"
    small = "gemm_tc3xf16_wgrad[M=28,N=1024,K=8192,splits=16,cluster=0,pair=0,bn=128]"
    timing = {big: (3.0, 60), small: (0.52, 20),
              "gemm_tc3xf16_fwd[M=8192,N=1024,K=1024,splits=1,cluster=0,pair=1,bn=128]": (2.8, 60)}
    pk = {"hbm_gbs": 6550.0, "bf16_tflops": 1650.0, "bf16_tflops_sustained": 1500.0}
    r = b.roofline(timing, pk, 1965.0, 20, "cfg4")
    assert r["launch"] == big and r["kernel"] == "gemm_tc3xf16_wgrad" and r["bound"] == "tensor"
    assert abs(r["achieved"] - 2 * 1024 * 1024 * 8192 / (3.0e-3 / 60) / 1e12) < 1e-3
    assert abs(r["peak"] - 1650.0 / 3) < 0.1  # three f16 MMAs per product against the f16 (= bf16) dense peak
    # traffic from the committed ncu capture of the kernel instance this launch ran: the split-K cluster (CLU) pair
    # kernel <BN, 3x, PAIR, MASK, F16, FAST, CLU, PART>
    tj = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
    if "cfg4:tc_gemm_kernel<128, 1, 1, 0, 1, 0, 1, 0>" in tj:
        assert r["traffic"] == tj["cfg4:tc_gemm_kernel<128, 1, 1, 0, 1, 0, 1, 0>"], r["traffic_source"]


def test_reference_arm_prints_one_json_line():
    """`--impl reference` times the oracle on host cores and prints the contract's line, alone on stdout."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "2", "--warmup", "3", "--cpu-budget", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env={**os.environ, "RANK": "0", "WORLD_SIZE": "1"})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 2 and d["warmup"] == 3
    assert d["unit"] == "samples/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["workload"].startswith("cfg4")  # the default workload: the largest config
    cb = d["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["nproc"] >= cb["cores"] and cb["cpu_model"]
