#!/bin/bash
# Round profile on the GPU box: tests-independent. Writes gpurun_out/prof/*.
# usage: bash tools/profile_round.sh <tag>
set -e
TAG=${1:-r1}
OUT=gpurun_out/prof
mkdir -p $OUT
python tools/bench_once.py 100 2 > $OUT/bench_once.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python tools/bench_once.py 100 2 > $OUT/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_sort_downsweep|k_sort_upsweep|k_fold_all|k_emit|k_seg_reduce|k_point_prep" \
    -s 36 -c 36 -o $OUT/${TAG}_full python tools/bench_once.py 100 2 > $OUT/ncu_full.log 2>&1
python bench.py --no-cpu-baseline > $OUT/bench_pre.json 2> $OUT/bench_pre.err
PASSES=$(python -c "import json; print(json.load(open('$OUT/bench_pre.json'))['work']['sort_passes'])")
python tools/summarize_profiles.py $TAG $OUT/${TAG}_launches.csv $OUT/${TAG}_full.ncu-rep $PASSES $OUT/bench_pre.json > $OUT/summary.log 2>&1
cp profiles/${TAG}_summary.md profiles/${TAG}_summary.json profiles/roofline_inputs.json $OUT/
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo done
