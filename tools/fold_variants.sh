# dev: apply-stage A/B of the long-run fold (window scan on/off, pairs per CTA)
for cfg in "1 0" "0 0" "1 3" "0 3"; do
  set -- $cfg
  VXG_FOLD_SCAN=$1 VXG_LONG_LAYOUT=$2 timeout 600 python bench.py --warmup 3 --steps 5 --no-cpu-baseline > gpurun_out/fv_$1_$2.json 2>gpurun_out/fv_$1_$2.err
  python -c "import json; d=json.load(open('gpurun_out/fv_$1_$2.json')); s=d['stages_ms_per_step']; print('scan $1 layout $2', round(d['ms_per_step'],3), 'apply', round(s['apply'],3), 'runs', round(s.get('runs',0),3), 'sort', round(s['record_sort'],3))"
  VXG_FOLD_SCAN=$1 VXG_LONG_LAYOUT=$2 VXG_FOLD_SERIAL=1 timeout 300 python tools/probe_fold.py 2>&1 | grep -v "^len"
done
