#!/bin/bash
# Round-2c final check on one B200: build + smoke, the GPU test suite, default bench line (cfg4, with the oracle's
# cpu_baseline), cfg2 line, the reference arm, then the cfg4 ncu launch list + --set full capture
set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.log 2>&1; tail -2 gpurun_out/final/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; tail -3 gpurun_out/final/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/final/bench_cfg4.json 2> gpurun_out/final/bench_cfg4.err; tail -2 gpurun_out/final/bench_cfg4.err
timeout 400 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/final/bench_cfg2.json 2> gpurun_out/final/bench_cfg2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
timeout 900 bash tools/ncu_capture.sh cfg4_r2c_final --steps 3 --warmup 3; echo ncu $?
