#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "3xf16" -p no:cacheprovider > gpurun_out/q_gemm.log 2>&1; tail -2 gpurun_out/q_gemm.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or cfg2" -p no:cacheprovider > gpurun_out/q_parity.log 2>&1; tail -2 gpurun_out/q_parity.log
for v in 1 0; do MTX_TC_BN256=$v timeout 300 python bench.py --no-cpu-baseline > gpurun_out/q_bench_bn256_$v.json 2> gpurun_out/q_bench_$v.err; done
python tools/show_bench.py -v gpurun_out/q_bench_bn256_1.json gpurun_out/q_bench_bn256_0.json
