mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r3h_bench_cfg1.json 2> gpurun_out/r3h_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r3h_bench_reference.json 2> gpurun_out/r3h_bench_reference.err; echo "ref rc=$?"
for c in 0 2 3; do timeout 600 python bench.py --config $c --steps 3 > gpurun_out/r3h_bench_cfg$c.json 2> gpurun_out/r3h_bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 900 python bench.py --config 4 --frames 8 --steps 2 > gpurun_out/r3h_bench_cfg4.json 2> gpurun_out/r3h_bench_cfg4.err; echo "cfg4 rc=$?"
timeout 300 python bench.py --gpus 1 --sharded-nccl --no-cpu-baseline --no-latency --steps 5 > gpurun_out/r3h_bench_cfg1_nccl1.json 2> gpurun_out/r3h_bench_cfg1_nccl1.err; echo "nccl1 rc=$?"
