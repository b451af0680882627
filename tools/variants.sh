for v in 1 2 4 5; do
  VXG_FOLD_SHORT_BLOCKS=$v timeout 600 python bench.py --warmup 3 --steps 5 --no-cpu-baseline > gpurun_out/bv$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bv$v.json')); s=d['stages_ms_per_step']; print('variant $v', round(d['ms_per_step'],3), 'apply', round(s['apply'],3), 'sort', round(s['record_sort'],3))"
done
