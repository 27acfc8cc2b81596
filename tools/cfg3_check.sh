#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 3xf16 3xtf32; do timeout 300 python bench.py --config cfg3 --precision $p --no-cpu-baseline > gpurun_out/cfg3_$p.json 2> gpurun_out/cfg3_$p.err; done
for p in 3xf16 3xtf32; do timeout 300 python bench.py --config cfg2 --precision $p --no-cpu-baseline > gpurun_out/cfg2_$p.json 2> gpurun_out/cfg2_$p.err; done
python tools/show_bench.py -v gpurun_out/cfg3_3xf16.json gpurun_out/cfg3_3xtf32.json gpurun_out/cfg2_3xf16.json gpurun_out/cfg2_3xtf32.json
