#!/bin/bash
# cfg2 3xTF32 step across builds of several commits ($BISECT) (tools/alt/<commit>, built here), same box.
mkdir -p gpurun_out/bis
for i in 1 2; do
  for c in ${BISECT:-old 92327f3 20b06f4 fb358c8}; do
    (cd tools/alt/$c && CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --config cfg2 --precision 3xtf32 --steps 50 --warmup 5 --no-cpu-baseline \
       > ../../../gpurun_out/bis/${c}_$i.json 2> ../../../gpurun_out/bis/${c}_$i.err)
  done
done
for f in gpurun_out/bis/*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['ms_per_step'], r['launches_us_per_step'])"; done
