#!/bin/bash
# quick A/B: cfg2 (3xTF32) and cfg4 (default) N=1 lines, twice each, plus the GEMM/step parity tests
mkdir -p gpurun_out/qb
for i in 1 2; do
  timeout 300 python bench.py --config cfg2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/qb/cfg2_$i.json 2> gpurun_out/qb/cfg2_$i.err
  timeout 300 python bench.py --config cfg4 --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/qb/cfg4_$i.json 2> gpurun_out/qb/cfg4_$i.err
done
for f in gpurun_out/qb/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['ms_per_step'], r['launches_us_per_step'])"; done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
