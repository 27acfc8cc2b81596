#!/bin/bash
# last check of the round's final commit on one B200: build + smoke, pytest -m gpu, default bench line
mkdir -p gpurun_out/last
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/last/smoke.log 2>&1; tail -1 gpurun_out/last/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/last/pytest_gpu.log 2>&1; tail -2 gpurun_out/last/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/last/bench_cfg4.json 2> gpurun_out/last/bench_cfg4.err
python tools/show_bench.py gpurun_out/last/bench_cfg4.json
