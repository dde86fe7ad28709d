#!/bin/bash
# One GPU cycle (run on the GPU box): parity suite, outdoor bench, serialised launch list.
# usage: scripts/gpu_cycle.sh TAG [extra pytest args]
tag=$1; shift
python -m pytest tests -m gpu -x -q "$@" > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --views 64 > gpurun_out/${tag}_ncu.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log
