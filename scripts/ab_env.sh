#!/bin/bash
# A/B of environment settings on the outdoor bench (quick: no e2e, no CPU baseline).
# usage: scripts/ab_env.sh out_prefix "NAME=VAR=VALUE[,VAR=VALUE]" ...   (run on the GPU box)
out=$1; shift
for spec in "$@"; do
  name=${spec%%=*}; envs=${spec#*=}
  env $(echo $envs | tr ',' ' ') python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} > ${out}_${name}.json 2> ${out}_${name}.err
  python -c "import json,sys; d=json.load(open('${out}_${name}.json')); print('$name', round(d['ms_per_step'],2), 'raster_own', round(d['serial_ms_per_step']['raster_ms'],2), 'front', round(d['serial_ms_per_step']['front_ms'],2), 'frac', round(d['roofline']['frac'],4))"
done
