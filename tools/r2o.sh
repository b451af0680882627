mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_free_functions.py tests/test_gpu_async_fold.py -x -q > gpurun_out/r2o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2o_pytest.log
timeout 120 python bench.py --no-latency --no-cpu-baseline --steps 5 > gpurun_out/r2o_bench_cfg1.json 2> gpurun_out/r2o_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r2o_bench_cfg0.json 2> gpurun_out/r2o_bench_cfg0.err; echo "cfg0 rc=$?"
timeout 200 python bench.py --config 2 --steps 3 --no-latency --no-cpu-baseline > gpurun_out/r2o_bench_cfg2.json 2> gpurun_out/r2o_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 200 python tools/probe_fold.py > gpurun_out/r2o_probe_fold.txt 2>&1
