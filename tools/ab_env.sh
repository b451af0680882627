#!/bin/bash
# A/B on the GPU box: one bench line per environment setting.
#   bash tools/ab_env.sh "" "VXG_FOLD_SHORT_BLOCKS=1" ...   ("" = defaults)
mkdir -p gpurun_out/ab
i=0
for setting in "$@"; do
  env $setting python bench.py --no-cpu-baseline > gpurun_out/ab/run_$i.json 2> gpurun_out/ab/run_$i.err
  echo "$setting" > gpurun_out/ab/run_$i.env
  i=$((i+1))
done
echo done
