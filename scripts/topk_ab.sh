#!/bin/bash
# A/B of library variants on the Eq. 6 finalize microbenchmark (scripts/bench_topk.py) at three
# row densities.   usage: scripts/topk_ab.sh out_prefix lib1.so [lib2.so ...]   (run on the GPU box)
out=$1; shift
for lib in "$@"; do
  name=$(basename $lib .so)
  for d in 0.0 0.3 1.0; do
    SCOUP_LIB=$lib python scripts/bench_topk.py 30 $d > ${out}_${name}_d${d}.json 2> ${out}_${name}_d${d}.err
    python -c "import json; d=json.load(open('${out}_${name}_d${d}.json')); print('$name', 'density', d['density'], 'ms', round(d['ms'],4), 'frac_hbm', round(d['frac_hbm'],3))"
  done
done
