#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 4 5 6 7; do echo "dbg $d"; MTX_TC_DBG=$d ENGINE=f16 SHAPES=0 python tools/gemm3x_bench.py 2>&1 | grep -E "tcts cta 0/|tcmma cta 0|\{" | tail -3; done > gpurun_out/tcts2.txt 2>&1
