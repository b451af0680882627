#!/bin/bash
# A/B of library builds on the GPU box: bash tools/ab_libs.sh tools/libvxg_a.so tools/libvxg_b.so ...
# ("default" = the in-tree build). One bench line per build in gpurun_out/ab/.
mkdir -p gpurun_out/ab
cp paper_1611_03631_b200/libvxg.so /tmp/libvxg_default.so
i=0
for lib in "$@"; do
  if [ "$lib" = default ]; then cp /tmp/libvxg_default.so paper_1611_03631_b200/libvxg.so; else cp "$lib" paper_1611_03631_b200/libvxg.so; fi
  python bench.py --no-cpu-baseline > gpurun_out/ab/run_$i.json 2> gpurun_out/ab/run_$i.err
  echo "$lib" > gpurun_out/ab/run_$i.env
  i=$((i+1))
done
cp /tmp/libvxg_default.so paper_1611_03631_b200/libvxg.so
echo done
