mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3j_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3j_pytest.log
timeout 200 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r3j_bench_cfg1.json 2> gpurun_out/r3j_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r3j_bench_cfg0.json 2> gpurun_out/r3j_bench_cfg0.err; echo "cfg0 rc=$?"
VXG_FOLD_PROD=2 timeout 200 python bench.py --config 2 --steps 3 --no-cpu-baseline --no-latency > gpurun_out/r3j_bench_cfg2_teams.json 2> gpurun_out/r3j_bench_cfg2.err; echo "cfg2 rc=$?"
