set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r2b_pytest.log
timeout 600 python bench.py > gpurun_out/r2b_bench_cfg1.json 2> gpurun_out/r2b_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --config 3 --steps 3 --no-latency --cpu-budget 5 > gpurun_out/r2b_bench_cfg3.json 2> gpurun_out/r2b_bench_cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config 4 --frames 8 --steps 3 --no-cpu-baseline --no-latency > gpurun_out/r2b_bench_cfg4.json 2> gpurun_out/r2b_bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo "ref rc=$?"
