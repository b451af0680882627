set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2c_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r2c_bench_cfg1.json 2> gpurun_out/r2c_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --config 3 --steps 3 --no-latency --cpu-budget 5 > gpurun_out/r2c_bench_cfg3.json 2> gpurun_out/r2c_bench_cfg3.err; echo "cfg3 rc=$?"
