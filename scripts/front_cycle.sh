#!/bin/bash
# GPU cycle for the front / Top-K kernels (run on the GPU box): parity suite, outdoor bench,
# serialised launch list, full ncu captures of the depth pass, the far predicate and the Top-K.
# usage: scripts/front_cycle.sh TAG [pytest -k expr]
tag=$1; k=${2:-}
if [ -n "$k" ]; then python -m pytest tests -m gpu -x -q -k "$k" > gpurun_out/${tag}_pytest.log 2>&1
else python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; fi; echo rc=$? >> gpurun_out/${tag}_pytest.log
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
python scripts/bench_topk.py 20 > gpurun_out/${tag}_topk.json 2>&1
python scripts/bench_topk.py 20 1.0 >> gpurun_out/${tag}_topk.json 2>&1
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --views 64 > gpurun_out/${tag}_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:depth_pass_kernel -s 2 -c 1 -o gpurun_out/${tag}_depth \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --views 32 > gpurun_out/${tag}_depth.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sel_count_kernel -s 2 -c 1 -o gpurun_out/${tag}_far \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --views 32 > gpurun_out/${tag}_far.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:topk_tile_kernel -s 1 -c 1 -o gpurun_out/${tag}_topk \
    python scripts/bench_topk.py 2 > gpurun_out/${tag}_topkncu.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
