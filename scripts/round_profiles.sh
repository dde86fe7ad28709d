#!/bin/bash
# The round's evidence (run on the GPU box): GPU suite, smoke, the default bench line (e2e and CPU
# baselines included), per-config lines, the serialised launch list of the bench command and a
# full ncu capture of the production raster launch.   usage: scripts/round_profiles.sh TAG
tag=$1
python -m pytest tests -m gpu -q > gpurun_out/${tag}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${tag}_pytest.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench_outdoor.json 2> gpurun_out/${tag}_bench_outdoor.err
for c in small indoor stress; do
  python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:raster2_kernel -s 2 -c 1 -o gpurun_out/${tag}_raster2 \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --views 16 > gpurun_out/${tag}_raster2.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
