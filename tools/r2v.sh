mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_mesh.py tests/test_gpu_sharded.py -x -q > gpurun_out/r2v_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2v_pytest.log
timeout 120 python bench.py --no-latency --no-cpu-baseline --steps 5 > gpurun_out/r2v_bench_cfg1.json 2> gpurun_out/r2v_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 300 python tools/probe_runs_cfg.py 4 1 > gpurun_out/r2v_runs_cfg4.txt 2>&1
timeout 300 python tools/probe_runs_cfg.py 3 100 > gpurun_out/r2v_runs_cfg3.txt 2>&1
timeout 300 python tools/probe_runs_cfg.py 2 50 > gpurun_out/r2v_runs_cfg2.txt 2>&1
