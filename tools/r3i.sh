mkdir -p gpurun_out
timeout 300 python tools/probe_f1.py 1 3 noprof > gpurun_out/r3i_f1_cfg1.txt 2>&1; echo "f1 rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_free_functions.py tests/test_gpu_async_fold.py tests/test_gpu_pipeline_env.py -x -q > gpurun_out/r3i_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3i_pytest.log
timeout 200 python tools/probe_fold.py > gpurun_out/r3i_probe.txt 2>&1
timeout 200 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r3i_bench_cfg1.json 2> gpurun_out/r3i_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r3i_bench_cfg0.json 2> gpurun_out/r3i_bench_cfg0.err; echo "cfg0 rc=$?"
timeout 200 python bench.py --config 2 --steps 3 --no-cpu-baseline --no-latency > gpurun_out/r3i_bench_cfg2.json 2> gpurun_out/r3i_bench_cfg2.err; echo "cfg2 rc=$?"
