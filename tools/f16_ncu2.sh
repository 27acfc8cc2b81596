#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 bash tools/ncu_capture.sh cfg4_f16 --precision 3xf16 --steps 3 --warmup 3; echo ncu $?
python tools/show_bench.py -v gpurun_out/ncu_plain_cfg4_f16.json
