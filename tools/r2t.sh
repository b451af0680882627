mkdir -p gpurun_out
bash tools/sanitize.sh r2t > gpurun_out/r2t_sanitize.out 2>&1
