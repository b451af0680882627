# A/B of the chunk pipeline on the GPU box: bench lines per VXG_CHUNK_RECORDS.
mkdir -p gpurun_out/ab
for v in default 134217728; do
  if [ $v = default ]; then unset VXG_CHUNK_RECORDS; else export VXG_CHUNK_RECORDS=$v; fi
  python bench.py --no-cpu-baseline > gpurun_out/ab/bench_$v.json 2> gpurun_out/ab/bench_$v.err
done
echo done
