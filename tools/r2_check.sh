#!/bin/bash
# Round-2 check on one B200: build + smoke, the GPU test suite, default (cfg4) and cfg2 bench lines,
# then the cfg4 ncu launch list + --set full capture (tools/ncu_capture.sh, after its plain run exits 0).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; tail -3 gpurun_out/bench_cfg4.err
timeout 400 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 bash tools/ncu_capture.sh ${NCU_TAG:-cfg4_final} --steps 3 --warmup 3; echo ncu $?
