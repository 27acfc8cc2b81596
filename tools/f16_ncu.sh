#!/bin/bash
# ncu --set full of the 3xF16 forward / dgrad / wgrad GEMMs at cfg4 shapes (tools/gemm3x_bench.py), one capture each
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ENGINE=f16 SHAPES=0,1,2 python tools/gemm3x_bench.py > gpurun_out/f16_ncu_plain.jsonl 2>&1 || exit 1
for sh in 0 1 2; do
  ENGINE=f16 SHAPES=$sh ncu --set full --clock-control none --import-source on -k "regex:tc_gemm_kernel" -s 4 -c 1 \
    -o gpurun_out/prof_f16_s$sh python tools/gemm3x_bench.py > gpurun_out/f16_ncu_s$sh.log 2>&1
done
SHAPES=0 ncu --set full --clock-control none -k "regex:tc_gemm_kernel" -s 4 -c 1 -o gpurun_out/prof_tf32_s0 python tools/gemm3x_bench.py > gpurun_out/tf32_ncu_s0.log 2>&1
echo done
