#!/bin/bash
# Summarise a GPU cycle's outputs here: scripts/show_cycle.sh TAG
tag=$1
tail -2 gpurun_out/${tag}_pytest.log
python -c "
import json; d=json.load(open('gpurun_out/${tag}_bench.json')); print('step', round(d['ms_per_step'],2), 'serial', {k: round(v,2) for k,v in d['serial_ms_per_step'].items()}, 'frac', round(d['roofline']['frac'],4), 'contrib', d['contributions_per_step'])"
python scripts/ncu_summary.py launches gpurun_out/${tag}_launches.csv | grep -v "at::\|red_kernel" | head -${2:-30}
