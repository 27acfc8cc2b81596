#!/bin/bash
# 3xF16 GEMM probe: cfg4 shapes at MTX_TC_DBG 0 (full) / 1 (no stores) / 2 (no loads) / 3 (MMA + drain only)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
out=gpurun_out/f16_probe${TAG}.jsonl
for d in ${DBGS:-0 1 2 3}; do MTX_TC_DBG=$d ENGINE=f16 SHAPES=${SH:-0,1,2,6,7,8} python tools/gemm3x_bench.py; done > $out 2>&1
