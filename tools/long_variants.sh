# dev: long-run fold layouts (serial = long runs alone)
for cfg in "0 0 0" "2 200000 148" "2 0 296" "2 0 444"; do
  set -- $cfg
  echo "layout $1 smem $2 ctas $3:"
  VXG_FOLD_SERIAL=1 VXG_LONG_LAYOUT=$1 VXG_LONG_SMEM=$2 VXG_LONG_CTAS=$3 python tools/probe_fold.py 2>&1 | sed -n 2,5p
done
