set -x
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2a_pytest.log
for c in 1 0 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2a_bench_cfg$c.json 2> gpurun_out/r2a_bench_cfg$c.err; echo "cfg$c rc=$?"
done
timeout 900 python bench.py --config 4 --frames 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_bench_cfg4.json 2> gpurun_out/r2a_bench_cfg4.err; echo "cfg4 rc=$?"
