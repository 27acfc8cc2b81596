#!/bin/bash
# A/B of the cfg2 3xTF32 step: commit 1ced31e (tools/alt/old, built here) vs the working tree, same box, interleaved.
mkdir -p gpurun_out/ab
for i in 1 2 3; do
  (cd tools/alt/old && timeout 300 python bench.py --config cfg2 --precision 3xtf32 --steps 50 --warmup 5 --no-cpu-baseline \
     > ../../../gpurun_out/ab/old_$i.json 2> ../../../gpurun_out/ab/old_$i.err)
  timeout 300 python bench.py --config cfg2 --precision 3xtf32 --steps 50 --warmup 5 --no-cpu-baseline \
     > gpurun_out/ab/new_$i.json 2> gpurun_out/ab/new_$i.err
done
for f in gpurun_out/ab/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['ms_per_step'], r['launches_us_per_step'])"; done
