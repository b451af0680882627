mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3r_launches_nccl1.csv python bench.py --gpus 1 --sharded-nccl --no-cpu-baseline --no-latency --steps 1 --warmup 3 > gpurun_out/r3r_ncu.log 2>&1; echo "ncu rc=$?"
