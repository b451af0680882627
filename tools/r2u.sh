mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2u_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2u_pytest.log
timeout 120 python bench.py --no-latency --no-cpu-baseline --steps 5 > gpurun_out/r2u_bench_cfg1.json 2> gpurun_out/r2u_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r2u_bench_cfg0.json 2> gpurun_out/r2u_bench_cfg0.err; echo "cfg0 rc=$?"
timeout 300 python bench.py --config 2 --steps 3 --no-latency --no-cpu-baseline > gpurun_out/r2u_bench_cfg2.json 2> gpurun_out/r2u_bench_cfg2.err; echo "cfg2 rc=$?"
timeout 300 python bench.py --config 3 --steps 3 --no-latency --no-cpu-baseline > gpurun_out/r2u_bench_cfg3.json 2> gpurun_out/r2u_bench_cfg3.err; echo "cfg3 rc=$?"
timeout 400 python bench.py --config 4 --frames 8 --steps 2 --no-latency --no-cpu-baseline > gpurun_out/r2u_bench_cfg4.json 2> gpurun_out/r2u_bench_cfg4.err; echo "cfg4 rc=$?"
