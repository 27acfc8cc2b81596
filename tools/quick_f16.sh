#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or cfg2" -p no:cacheprovider > gpurun_out/q_parity.log 2>&1; tail -2 gpurun_out/q_parity.log
for p in 3xf16; do timeout 300 python bench.py --precision $p --no-cpu-baseline > gpurun_out/q_bench_$p.json 2> gpurun_out/q_bench_$p.err; done
python tools/show_bench.py -v gpurun_out/q_bench_3xf16.json
