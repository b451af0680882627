# Round-end measurement on the GPU box: full GPU suite, smoke, profile round (launch list + --set full),
# bench lines of every config, the 1-rank NCCL line and the fold trace. Usage: gpurun -- bash tools/final_round.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"
rm -rf gpurun_out/prof; timeout 1800 bash tools/profile_round.sh r3 > gpurun_out/final_profile.log 2>&1; echo "profile rc=$?"
for c in 0 2 3; do timeout 600 python bench.py --config $c --steps 3 > gpurun_out/final_bench_cfg$c.json 2> gpurun_out/final_bench_cfg$c.err; echo "cfg$c rc=$?"; done
timeout 900 python bench.py --config 4 --frames 8 --steps 2 > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err; echo "cfg4 rc=$?"
timeout 300 python bench.py --gpus 1 --sharded-nccl --no-cpu-baseline --no-latency --steps 5 > gpurun_out/final_bench_cfg1_nccl1.json 2> gpurun_out/final_bench_cfg1_nccl1.err; echo "nccl1 rc=$?"
timeout 200 python tools/probe_fold.py > gpurun_out/final_probe.txt 2>&1
