#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cmd="python bench.py --precision 3xf16 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --set full --import-source on --clock-control none -k "regex:fwd_smallk" -s 2 -c 1 --warp-sampling-interval 0 -o gpurun_out/prof_f16_small $cmd > gpurun_out/f16_ncu4.log 2>&1
echo done $?
