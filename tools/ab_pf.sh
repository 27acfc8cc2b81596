#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for pf in 0 4 8; do MTX_TC_PF=$pf timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_pf$pf.json 2>/dev/null; done
python tools/show_bench.py -v gpurun_out/ab_pf0.json gpurun_out/ab_pf4.json gpurun_out/ab_pf8.json
