mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_free_functions.py tests/test_gpu_async_fold.py -x -q > gpurun_out/r2r_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2r_pytest.log
timeout 200 python tools/probe_fold.py > gpurun_out/r2r_probe.txt 2>&1
VXG_FOLD_MERGED=0 VXG_FOLD_SERIAL=1 timeout 200 python tools/probe_fold.py > gpurun_out/r2r_probe_serial.txt 2>&1
timeout 120 python bench.py --no-latency --no-cpu-baseline --steps 5 > gpurun_out/r2r_bench_cfg1.json 2> gpurun_out/r2r_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r2r_bench_cfg0.json 2> gpurun_out/r2r_bench_cfg0.err; echo "cfg0 rc=$?"
