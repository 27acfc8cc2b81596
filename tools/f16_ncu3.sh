#!/bin/bash
# one in-step forward and dgrad GEMM of cfg4 3xF16 with fine warp-state sampling (source page)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cmd="python bench.py --precision 3xf16 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --set full --import-source on --warp-sampling-interval 0 --clock-control none -k regex:tc_gemm_kernel -s 40 -c 6 -o gpurun_out/prof_f16_step $cmd > gpurun_out/f16_ncu3.log 2>&1
echo done $?
