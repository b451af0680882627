mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2n_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2n_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2n_smoke.log 2>&1; echo "smoke rc=$?"
timeout 400 python bench.py > gpurun_out/r2n_bench_cfg1.json 2> gpurun_out/r2n_bench_cfg1.err; echo "cfg1 rc=$?"
timeout 400 python bench.py --impl reference > gpurun_out/r2n_bench_reference.json 2> gpurun_out/r2n_bench_reference.err; echo "ref rc=$?"
