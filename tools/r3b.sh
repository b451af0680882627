mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_mesh.py tests/test_gpu_sharded.py -x -q > gpurun_out/r3b_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3b_pytest.log
timeout 120 python bench.py --no-latency --no-cpu-baseline --steps 5 > gpurun_out/r3b_bench_cfg1.json 2> gpurun_out/r3b_bench_cfg1.err; echo "cfg1 rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b_launches.csv python tools/bench_once.py 100 2 > gpurun_out/r3b_ncu.log 2>&1; echo "ncu rc=$?"
