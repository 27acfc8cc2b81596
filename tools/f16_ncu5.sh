#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cmd="python bench.py --precision 3xf16 --steps 2 --warmup 3 --no-cpu-baseline"
ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel -s 30 -c 10 -o gpurun_out/prof_f16_step2 $cmd > gpurun_out/f16_ncu5.log 2>&1
echo done $?
