mkdir -p gpurun_out/ab
cp paper_1611_03631_b200/libvxg.so /tmp/libvxg_default.so
i=0
for lib in default tools/libvxg_reg96.so tools/libvxg_reg80.so tools/libvxg_reg64.so default; do
  if [ "$lib" = default ]; then cp /tmp/libvxg_default.so paper_1611_03631_b200/libvxg.so; else cp "$lib" paper_1611_03631_b200/libvxg.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-latency --steps 8 > gpurun_out/ab/k_$i.json 2> gpurun_out/ab/k_$i.err
  echo "$lib" > gpurun_out/ab/k_$i.env
  i=$((i+1))
done
cp /tmp/libvxg_default.so paper_1611_03631_b200/libvxg.so
