mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3f_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r3f_pytest.log
timeout 200 python tools/probe_f1.py 0 4 > gpurun_out/r3f_f1_cfg0.txt 2>&1
timeout 200 python tools/probe_f1.py 1 4 > gpurun_out/r3f_f1_cfg1.txt 2>&1
VXG_FIXED_LONG_RUN=1 timeout 200 python tools/probe_f1.py 1 4 > gpurun_out/r3f_f1_cfg1_fixed.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r3f_bench_cfg1.json 2> gpurun_out/r3f_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 120 python bench.py --config 0 --steps 3 --no-cpu-baseline > gpurun_out/r3f_bench_cfg0.json 2> gpurun_out/r3f_bench_cfg0.err; echo "cfg0 rc=$?"
