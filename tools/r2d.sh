set -x
python -m pytest tests/test_gpu_sharded.py tests/test_gpu_parity.py -x -q > gpurun_out/r2d_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2d_pytest.log
timeout 900 python bench.py --config 3 --steps 3 --no-latency --cpu-budget 5 > gpurun_out/r2d_bench_cfg3.json 2> gpurun_out/r2d_bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --sharded-nccl --steps 5 --no-latency --no-cpu-baseline > gpurun_out/r2d_bench_cfg1_nccl1.json 2> gpurun_out/r2d_bench_cfg1_nccl1.err; echo "nccl1 rc=$?"
