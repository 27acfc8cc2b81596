#!/bin/bash
# Usage (on the GPU box, one GPU): tools/ncu_capture.sh <tag> <bench args...>
# 1) the plain command must exit 0;  2) launch list (every kernel's device time);
# 3) one --set full capture of the dominant kernels.  Outputs in gpurun_out/.
set -e
tag=$1; shift
cmd="python bench.py $* --no-cpu-baseline"
$cmd > gpurun_out/ncu_plain_$tag.json 2> gpurun_out/ncu_plain_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv $cmd > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k "regex:tc_gemm_kernel|avg_update|head_kernel|gemm_simt|conv_|colsum|fwd_smallk|quantize_f16|wgrad_narrow" -s 40 -c 12 -o gpurun_out/prof_$tag $cmd > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu done $tag"
