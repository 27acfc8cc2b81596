#!/bin/bash
# build, smoke, single-GPU tests, and the bench lines for cfg2/cfg4 (3xtf32 + tf32) with a compact summary
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q -k "not multigpu" -x > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
grep -E "^E  +(Assertion|assert)" gpurun_out/pytest_gpu.log | head -4
for c in ${CONFIGS:-cfg2 cfg4}; do for p in ${PRECS:-3xtf32 tf32}; do
  timeout 300 python bench.py --config $c --precision $p --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${c}_$p.json 2>gpurun_out/bench_${c}_$p.err || tail -3 gpurun_out/bench_${c}_$p.err
  python tools/show_bench.py gpurun_out/bench_${c}_$p.json
done; done
