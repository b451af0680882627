mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_async_fold.py tests/test_gpu_pipeline_env.py -x -q > gpurun_out/r3n_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3n_pytest.log
timeout 200 python bench.py --no-cpu-baseline --no-latency --steps 8 > gpurun_out/r3n_bench_cfg1.json 2> gpurun_out/r3n_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 300 python bench.py --config 3 --steps 3 --no-cpu-baseline --no-latency > gpurun_out/r3n_bench_cfg3.json 2> gpurun_out/r3n_bench_cfg3.err; echo "cfg3 rc=$?"
timeout 300 python bench.py --config 2 --steps 3 --no-cpu-baseline --no-latency > gpurun_out/r3n_bench_cfg2.json 2> gpurun_out/r3n_bench_cfg2.err; echo "cfg2 rc=$?"
