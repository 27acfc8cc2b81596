#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MTX_TC_DBG=4 ENGINE=f16 SHAPES=0,6,2 python tools/gemm3x_bench.py > gpurun_out/tcts_probe.txt 2>&1
MTX_TC_DBG=4 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tcts_bench.json 2> gpurun_out/tcts_bench.err
grep tcts gpurun_out/tcts_bench.json gpurun_out/tcts_bench.err | tail -40 > gpurun_out/tcts_step.txt
