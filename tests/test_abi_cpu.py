"""CPU-side checks of the boundary: libmtx.so loads, exports every function
include/mtx.h declares, and its pure host helper (mtx_batch_slice) agrees with
the oracle's shard rule.  No compute calls (no GPU here)."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "mtx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mtx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["mtx_init", "mtx_bcast_params", "mtx_shard_data", "mtx_train_step", "mtx_allreduce_avg"]:
        assert n in names  # BASELINE.json north_star's C-ABI


def test_library_exports_every_declared_symbol():
    from paper_1704_04560_b200 import build
    lib = build.build()
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (mtx_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    h = ctypes.CDLL(lib)
    for n in declared():
        getattr(h, n)


def test_library_is_sm100a():
    from paper_1704_04560_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_batch_slice_matches_oracle():
    from paper_1704_04560_b200 import mtx
    for n in (10, 100, 1000, 60000):
        for P in (1, 2, 4, 8):
            for B in (8, 64, 512):
                if B > n or B % P:
                    continue
                for step in (0, 1, 13, 117, 10 ** 9):
                    for r in range(P):
                        assert mtx.mtx_batch_slice(n, B, step, r, P) == oracle.batch_slice(n, B, step, r, P)
    with pytest.raises(mtx.MtxError):
        mtx.mtx_batch_slice(100, 6, 0, 0, 4)
    with pytest.raises(mtx.MtxError):
        mtx.mtx_batch_slice(4, 8, 0, 0, 1)


def test_build_entry_does_not_need_the_library(tmp_path):
    """__graft_entry__.build() runs in a fresh checkout, before libmtx.so exists: loading the
    builder must not import the package (whose import loads the library)."""
    code = (
        "import sys, __graft_entry__ as g, importlib.util, os\n"
        "spec = importlib.util.spec_from_file_location('_b', os.path.join(g.ROOT, 'paper_1704_04560_b200', 'build.py'))\n"
        "b = importlib.util.module_from_spec(spec); spec.loader.exec_module(b)\n"
        "assert callable(b.build)\n"
        "assert 'paper_1704_04560_b200' not in sys.modules, 'builder imported the package'\n"
        "import inspect\n"
        "src = inspect.getsource(g.build)\n"
        "assert src.index('b.build()') < src.index('import paper_1704_04560_b200'), 'package imported before build'\n"
        "assert 'from paper_1704_04560_b200' not in src\n")
    subprocess.run(["python", "-c", code], cwd=ROOT, check=True)


def test_tf32_is_not_a_product_precision():
    """Reading A22: mtx_init refuses MTX_TF32 (1xTF32 cannot meet the north_star's 1e-3) unless the development
    variable is set; the check precedes any CUDA call, so it runs on a CPU host."""
    import mtx_synth as S
    from paper_1704_04560_b200 import mtx
    if os.environ.get("MTX_DEV_TF32"):
        pytest.skip("development override set")
    cfg = S.CONFIGS["cfg1"]
    with pytest.raises(mtx.MtxError) as e:
        mtx.mtx_init(0, 1, None, 0, mtx.model_desc(cfg, 64), mtx.optim_desc(0.1, 0.0, mtx.MTX_TF32, 0, 0, 42))
    assert e.value.status == 9  # MTX_ERR_UNSUPPORTED
