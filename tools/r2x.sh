mkdir -p gpurun_out
python tools/bench_once.py 100 2 > gpurun_out/r2x_once.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_launches.csv python tools/bench_once.py 100 2 > gpurun_out/r2x_ncu.log 2>&1; echo "ncu rc=$?"
