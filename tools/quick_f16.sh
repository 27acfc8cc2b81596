#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
DBGS=0 SH=0,1,2,9,10 TAG=_q bash tools/f16_probe.sh
MTX_TC_BN=128 ENGINE=f16 SHAPES=9 python tools/gemm3x_bench.py >> gpurun_out/f16_probe_q.jsonl 2>&1
MTX_TC_BN=64 ENGINE=f16 SHAPES=9 python tools/gemm3x_bench.py >> gpurun_out/f16_probe_q.jsonl 2>&1
for p in 3xf16; do timeout 300 python bench.py --precision $p --no-cpu-baseline > gpurun_out/q_bench_$p.json 2> gpurun_out/q_bench_$p.err; done
python tools/show_bench.py -v gpurun_out/q_bench_3xf16.json
