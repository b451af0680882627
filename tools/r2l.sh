mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fold_all" -s 3 -c 1 \
   -o gpurun_out/prof/r2l_fold_cfg4 python tools/bench_cfg_once.py 4 4 1 > gpurun_out/prof/r2l_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/r2l_launches_cfg4.csv python tools/bench_cfg_once.py 4 4 1 > /dev/null 2>&1; echo "launch rc=$?"
