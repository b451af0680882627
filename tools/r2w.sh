mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fold_all -c 2 -o gpurun_out/r2w_fold_cfg4 python tools/bench_cfg_once.py 4 1 1 > gpurun_out/r2w_ncu.log 2>&1; echo "ncu rc=$?"
