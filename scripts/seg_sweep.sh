#!/bin/bash
# Sweep of the binning sort's forced segment length on one bench config (quick: no e2e, no CPU
# baseline).   usage: scripts/seg_sweep.sh out_prefix config len1 [len2 ...]   (0 = adaptive)
out=$1; cfg=$2; shift; shift
for n in "$@"; do
  python -c "
import runpy, sys
from paper_2605_13600_b200 import abi
abi.scoup_diag_set_binsort_segment($n)
sys.argv = ['bench.py', '--config', '$cfg', '--steps', '2', '--warmup', '3', '--no-e2e', '--no-cpu-baseline'] + '${AB_ARGS}'.split()
runpy.run_path('bench.py', run_name='__main__')" > ${out}_seg${n}.json 2> ${out}_seg${n}.err
  python -c "import json; d=json.load(open('${out}_seg${n}.json')); print('seg $n', round(d['ms_per_step'],2), 'raster_own', round(d['serial_ms_per_step']['raster_ms'],2), 'front', round(d['serial_ms_per_step']['front_ms'],2))"
done
