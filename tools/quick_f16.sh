#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg4 or cfg2 or head" -p no:cacheprovider > gpurun_out/q_parity.log 2>&1; tail -2 gpurun_out/q_parity.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err

python tools/show_bench.py -v gpurun_out/q_bench.json
