mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sharded.py -x -q > gpurun_out/r3q_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r3q_pytest.log
timeout 300 python bench.py --gpus 1 --sharded-nccl --no-cpu-baseline --no-latency --steps 5 > gpurun_out/r3q_bench_cfg1_nccl1.json 2> gpurun_out/r3q_bench_cfg1_nccl1.err; echo "nccl1 rc=$?"
